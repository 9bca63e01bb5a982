mkdir -p gpurun_out
T0=$(date +%s)
timeout 1200 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "rc=$? wall=$(( $(date +%s) - T0 ))s"; tail -2 gpurun_out/bench_default.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_default.json").read().strip().splitlines()[-1])
print({k: d[k] for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling", "vs_baseline", "dtype", "gpu_launches")})
print("e2e", round(d["e2e"]["value"] / 1e9, 2), "roofline", round(d["roofline"]["frac"], 3), "cpu", d["cpu_baseline"]["value"])
PY
timeout 1200 python bench.py --impl reference --gpus 1 --steps 5 --warmup 3 > gpurun_out/bench_ref_default.json 2> gpurun_out/bench_ref_default.err; echo "ref rc=$?"; tail -1 gpurun_out/bench_ref_default.err; tail -c 300 gpurun_out/bench_ref_default.json
