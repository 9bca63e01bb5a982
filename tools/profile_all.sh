#!/bin/bash
# Run on the GPU box (gpurun): plain run then ncu --set full of lx_rollout (at the
# bench batch, 2^22 envs, so per-env-step counts match the bench workload) for
# each config game, SASS source pages exported, plus the bench launch list.
mkdir -p gpurun_out
for gb in ${GAMES:-connect_four:4194304 tic_tac_toe:4194304 hex:4194304 reversi:4194304 pente:4194304}; do
  g=${gb%%:*}; b=${gb##*:}
  timeout 300 python tools/ncu_rollout.py --game $g --batch $b > gpurun_out/plain_$g.json 2>&1 &&
  timeout 600 ncu --set full --metrics sm__inst_executed_pipe_alu.sum,sm__inst_executed_pipe_alu.avg.peak_sustained,sm__cycles_elapsed.avg \
      --clock-control none --import-source on -k regex:"^lx_rollout$" -s 1 -c 1 \
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
# per-ply HBM-bound kernels (bench.py `traffic` of step_kernel / env_step_api)
for gb in ${STEP_GAMES:-}; do
  g=${gb%%:*}; b=${gb##*:}
  timeout 300 python tools/ncu_step.py --game $g --batch $b > gpurun_out/step_$g.json 2>&1 || continue
  for ks in lx_random_step:2:lx_random_step lx_env_step:3:lx_env_step lx_env_step:8:lx_env_step_bits; do
    k=${ks%%:*}; rest=${ks#*:}; skip=${rest%%:*}; tag=${rest#*:}
    timeout 300 ncu --set full --clock-control none -k regex:"^$k\$" -s $skip -c 1 \
        -o gpurun_out/stepprof_${g}_$tag python tools/ncu_step.py --game $g --batch $b \
        > gpurun_out/ncu_step_${g}_$tag.log 2>&1
    echo "$g $tag rc=$?"
  done
done
