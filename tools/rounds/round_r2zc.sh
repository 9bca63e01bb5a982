# cluster publish for 2..8-block rollout grids: tests + latency A/B (same build, host switch)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_playout_host.py tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_c_abi.py -m gpu -q -x > gpurun_out/pytest_cluster.log 2>&1; tail -3 gpurun_out/pytest_cluster.log
for B in 1024 2048 512; do
  timeout 300 python tools/latency_probe.py --game tic_tac_toe --batch $B --caps 0,200 2>&1 | grep -v trivial
  LX_NO_CLUSTER_LAUNCH=1 timeout 300 python tools/latency_probe.py --game tic_tac_toe --batch $B --caps 0,200 2>&1 | grep -v trivial | sed 's/"variant": {}/"variant": {"LX_NO_CLUSTER_LAUNCH": "1"}/'
done > gpurun_out/lat_cluster.jsonl
cat gpurun_out/lat_cluster.jsonl
for g in connect_four pente tic_tac_toe hex reversi; do
  timeout 300 python tools/ab_env.py --game $g --reps 8 --variant "" --variant LX_PUBLISH_INLINE=1 --variant LX_PUBLISH_INLINE=0 >> gpurun_out/ab_r2zc.jsonl 2>>gpurun_out/ab_r2zc.err
done
python - <<'PY'
import json
for line in open("gpurun_out/ab_r2zc.jsonl"):
    d = json.loads(line)
    print(d["game"], d["same_stats"], [(v["env"], round(v["env_steps_per_s"] / 1e9, 2)) for v in d["variants"]])
PY
