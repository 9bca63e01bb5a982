# r2r: converged reach-set flood in lx_rollout (split ply), A/B + Hex/Yavalath parity
mkdir -p gpurun_out
timeout 600 python tools/ab_env.py --game hex --reps 10 --variant LX_SPLIT_FLOOD=0 --variant "" > gpurun_out/ab_r2r.jsonl 2> gpurun_out/ab_r2r.err
timeout 600 python tools/ab_env.py --game yavalath --reps 10 --variant LX_SPLIT_FLOOD=0 --variant "" >> gpurun_out/ab_r2r.jsonl 2>> gpurun_out/ab_r2r.err
python - <<'PY'
import json
for line in open("gpurun_out/ab_r2r.jsonl"):
    d = json.loads(line)
    print(d["game"], d["same_stats"], [(v["env"], round(v["env_steps_per_s"] / 1e9, 2)) for v in d["variants"]])
PY
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py -q -x -k "hex or yavalath or full_size or work_buffer or host_edits" > gpurun_out/pytest_r2r.log 2>&1; tail -3 gpurun_out/pytest_r2r.log
