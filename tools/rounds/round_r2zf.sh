# async host-buffer pipeline: tests + bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_playout_host.py tests/test_c_abi.py -m gpu -q -x > gpurun_out/pytest_async.log 2>&1; tail -3 gpurun_out/pytest_async.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench rc=$?"; tail -c 300 gpurun_out/bench_c4.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_c4.json").read().strip().splitlines()[-1])
print("head", round(d["value"]/1e9,2), "e2e", round(d["e2e"]["value"]/1e9,2), "e2e_c_abi", round(d.get("e2e_c_abi",{}).get("value",0)/1e9,2))
for c in d.get("per_config", []):
    e = c.get("e2e"); h = c.get("e2e_c_abi")
    print(c["config"], round(c["value"]/1e9,3), e if isinstance(e,str) else round(e["value"]/1e9,3), round(h["value"]/1e9,3) if isinstance(h,dict) else h)
PY
