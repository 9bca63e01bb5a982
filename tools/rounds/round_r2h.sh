# r2h: row mirror for Pente (shared-memory row planes, 128-thread blocks), Reversi
# shifts on the FMA pipe: GPU suite, A/B, bench
mkdir -p gpurun_out
timeout 600 python tools/ab_env.py --game pente --reps 6 --variant LX_ROW_MIRROR=0 --variant "" > gpurun_out/ab_r2h.jsonl 2> gpurun_out/ab_r2h.err
timeout 600 python tools/ab_env.py --game reversi --reps 10 --variant LX_SHIFT_FMA=0 --variant "" >> gpurun_out/ab_r2h.jsonl 2>> gpurun_out/ab_r2h.err
python - <<'PY'
import json
for line in open("gpurun_out/ab_r2h.jsonl"):
    d = json.loads(line)
    print(d["game"], d["same_stats"], [(v["env"], round(v["env_steps_per_s"] / 1e9, 2)) for v in d["variants"]])
PY
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -6 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench rc=$?"; tail -c 300 gpurun_out/bench_c4.err
