# r2f: self-clearing rollout work buffer (no memsets), unroll/SWAR/place_bit build:
# GPU suite, ncu of the five config games (rollout + step kernels), bench (after
# the captures, so the roofline reads this build's counts), sweep, reference arm.
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -4 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -3 gpurun_out/smoke.log
NO_LAUNCHES=1 STEP_GAMES="connect_four:4194304 tic_tac_toe:4194304 hex:4194304 reversi:4194304 pente:4194304" bash tools/profile_all.sh
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench rc=$?"; tail -c 300 gpurun_out/bench_c4.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout 900 python tools/sweep.py --min-log2 10 --max-log2 22 > gpurun_out/sweep.jsonl 2> gpurun_out/sweep.err; echo "sweep rc=$?"
timeout 300 python bench.py --steps 3 --warmup 1 --no-extras > gpurun_out/b_plain.log 2>&1 && timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 1 --no-extras > gpurun_out/ncu_launch.log 2>&1; echo "launches rc=$?"
