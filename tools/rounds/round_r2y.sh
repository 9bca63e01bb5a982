mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_playout_host.py tests/test_c_abi.py -m gpu -q -x > gpurun_out/pytest_playout.log 2>&1; tail -3 gpurun_out/pytest_playout.log
timeout 300 python tools/probe_playout_host.py > gpurun_out/probe_ph.jsonl 2>&1; tail -1 gpurun_out/probe_ph.jsonl
LX_PLAYOUT_FIRST_PIECE=65536 LX_PLAYOUT_MAX_PIECE=65536 timeout 300 python tools/probe_playout_host.py 2>&1 | tail -1
LX_PLAYOUT_FIRST_PIECE=262144 LX_PLAYOUT_MAX_PIECE=1048576 timeout 300 python tools/probe_playout_host.py 2>&1 | tail -1
LX_PLAYOUT_FIRST_PIECE=4096 LX_PLAYOUT_MAX_PIECE=4194304 timeout 300 python tools/probe_playout_host.py 2>&1 | tail -1
timeout 300 python tools/probe_playout_host.py --game tic_tac_toe 2>&1 | tail -1
timeout 300 python tools/probe_playout_host.py --game hex 2>&1 | tail -1
for g in pente connect_four hex; do
  timeout 300 python tools/ab_env.py --game $g --reps 8 --variant "" --variant "LX_STATIC_CHUNKS=0,LX_ACQREL_TICKET=0" >> gpurun_out/ab_r2y.jsonl 2>>gpurun_out/ab_r2y.err
done
python - <<'PY'
import json
for line in open("gpurun_out/ab_r2y.jsonl"):
    d = json.loads(line)
    print(d["game"], d["same_stats"], [(v["env"], round(v["env_steps_per_s"] / 1e9, 2)) for v in d["variants"]])
PY
