# packed single-copy export + read-only planes: full GPU suite + bench
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -6 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench rc=$?"; tail -c 300 gpurun_out/bench_c4.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_c4.json").read().strip().splitlines()[-1])
print("head", round(d["value"]/1e9,2), "e2e", round(d["e2e"]["value"]/1e9,2), "e2e_python", round(d["e2e_python"]["value"]/1e9,2), "ref_layout", d.get("e2e_reference_layout"))
PY
