# r2d: full GPU suite; ncu of lx_rollout (5 config games, with SASS source
# pages) and of the per-ply kernels (random step, env step bool / bits); bench.
mkdir -p gpurun_out
timeout 2000 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -15 gpurun_out/pytest_gpu.log
tail -5 gpurun_out/ref_test_engine_over_adapter.log gpurun_out/ref_test_acceptance_over_adapter.log
NO_LAUNCHES=1 STEP_GAMES="connect_four:4194304 tic_tac_toe:4194304 hex:4194304 reversi:4194304 pente:4194304" bash tools/profile_all.sh
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench rc=$?"; tail -c 300 gpurun_out/bench_c4.err
timeout 300 python bench.py --steps 3 --warmup 1 --no-extras > gpurun_out/b_plain.log 2>&1 && timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 1 --no-extras > gpurun_out/ncu_launch.log 2>&1; echo "launches rc=$?"
