mkdir -p gpurun_out
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench rc=$?"; tail -c 600 gpurun_out/bench_c4.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_c4.json").read().strip().splitlines()[-1])
print("head", round(d["value"]/1e9,2), "e2e", round(d["e2e"]["value"]/1e9,2), d["e2e"].get("roofline"))
print("e2e_python", round(d["e2e_python"]["value"]/1e9,2), d["e2e_python"].get("roofline"))
for c in d.get("per_config", []):
    e = c.get("e2e")
    if isinstance(e, dict): print(c["config"], round(e["value"]/1e9,3), {k: round(v,3) if isinstance(v,float) else v for k,v in (e.get("roofline") or {}).items() if k in ("achieved","peak","frac","bound_env_steps_per_s")})
PY
