# r1r: ncu --set full of the per-ply HBM-bound kernels (lx_random_step, lx_sample,
# lx_env_step) for the five config games, summaries written on the box so the
# bench line carries their DRAM traffic; then the C4 bench.
mkdir -p gpurun_out/profiles
for gb in connect_four:4194304 tic_tac_toe:4194304 hex:4194304 reversi:4194304 pente:4194304; do
  g=${gb%%:*}; b=${gb##*:}
  timeout 300 python tools/ncu_step.py --game $g --batch $b > gpurun_out/step_$g.json 2>&1 || { tail -3 gpurun_out/step_$g.json; continue; }
  for k in lx_random_step lx_sample lx_env_step; do
    timeout 300 ncu --set full --clock-control none -k regex:"^$k\$" -s 2 -c 1 \
        -o gpurun_out/stepprof_${g}_$k python tools/ncu_step.py --game $g --batch $b \
        > gpurun_out/ncu_step_${g}_$k.log 2>&1
    echo "$g $k rc=$?"
  done
done
python tools/ncu_summary.py gpurun_out --tag r1r > gpurun_out/summary.log 2>&1; cat gpurun_out/summary.log
cp profiles/r1r_step_* profiles/step_*.json gpurun_out/profiles/
python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; tail -c 1200 gpurun_out/bench_c4.json
