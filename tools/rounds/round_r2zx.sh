mkdir -p gpurun_out
for i in 1 2 3; do
timeout 900 python bench.py --steps 20 --warmup 5 --no-per-config > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_c4.json").read().strip().splitlines()[-1])
print("head", round(d["value"]/1e9,2), "e2e", round(d["e2e"]["value"]/1e9,2), "e2e_python", round(d["e2e_python"]["value"]/1e9,2), "pcie", round(d["e2e"]["roofline"]["pcie_h2d"]["peak_gbs"],1))
PY
done
