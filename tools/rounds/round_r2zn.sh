mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_reference_driver.py tests/test_gpu_env.py tests/test_gpu_playout_host.py -m gpu -q -x > gpurun_out/pytest_sub.log 2>&1; tail -3 gpurun_out/pytest_sub.log
timeout 900 python bench.py --steps 20 --warmup 5 --no-per-config > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench rc=$?"; tail -c 300 gpurun_out/bench_c4.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_c4.json").read().strip().splitlines()[-1])
print("head", round(d["value"]/1e9,2), "e2e", round(d["e2e"]["value"]/1e9,2), "e2e_python", round(d["e2e_python"]["value"]/1e9,2), "ref_layout", round(d["e2e_reference_layout"]["value"]/1e9, 3))
PY
timeout 600 python tools/mcts_bench.py --game connect_four --games 16 --no-reference 2>&1 | tail -c 200
timeout 300 python tools/probe_playout_host.py --game tic_tac_toe --batch 1024 --reps 300 2>&1 | tail -1
