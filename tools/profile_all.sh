#!/bin/bash
# Run on the GPU box (gpurun): plain run then ncu --set full of lx_rollout for
# each config game, SASS source pages exported, plus the bench launch list.
mkdir -p gpurun_out
for gb in ${GAMES:-connect_four:1048576 tic_tac_toe:1048576 hex:131072 reversi:262144 pente:65536}; do
  g=${gb%%:*}; b=${gb##*:}
  timeout 300 python tools/ncu_rollout.py --game $g --batch $b > gpurun_out/plain_$g.json 2>&1 &&
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:lx_rollout -s 1 -c 1 \
      -o gpurun_out/prof_$g python tools/ncu_rollout.py --game $g --batch $b > gpurun_out/ncu_$g.log 2>&1
  echo "$g rc=$?"
  ncu -i gpurun_out/prof_$g.ncu-rep --page source --csv --print-source sass > gpurun_out/sass_$g.csv 2>/dev/null
done
if [ -z "$NO_LAUNCHES" ]; then
  timeout 300 python bench.py --steps 3 --warmup 1 --no-extras > gpurun_out/b_plain.log 2>&1 &&
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
      --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 1 --no-extras > gpurun_out/ncu_launch.log 2>&1
  echo "launches rc=$?"
fi
