# small-grid rollout start/publish A/B (static chunks, acq_rel ticket) + occupancy variants
mkdir -p gpurun_out
OLD=LX_STATIC_CHUNKS=0,LX_ACQREL_TICKET=0
for B in 1024 32 8192; do
  for v in "" "$OLD" "LX_ACQREL_TICKET=0"; do
    timeout 300 python tools/latency_probe.py --game tic_tac_toe --batch $B --caps 0,200 --variant "$v" 2>&1 | grep -v trivial
  done
done > gpurun_out/lat_ab.jsonl 2>&1
timeout 300 python tools/latency_probe.py --game connect_four --batch 1024 --caps 0,200 >> gpurun_out/lat_ab.jsonl 2>&1
timeout 300 python tools/latency_probe.py --game connect_four --batch 1024 --caps 0,200 --variant "$OLD" >> gpurun_out/lat_ab.jsonl 2>&1
cat gpurun_out/lat_ab.jsonl
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py -m gpu -q -x > gpurun_out/pytest_sub.log 2>&1; tail -2 gpurun_out/pytest_sub.log
for g in connect_four tic_tac_toe hex; do
  timeout 300 python tools/ab_env.py --game $g --reps 10 --variant "" --variant "$OLD" >> gpurun_out/ab_r2v.jsonl 2>>gpurun_out/ab_r2v.err
done
timeout 300 python tools/ab_env.py --game reversi --reps 10 --variant "" --variant "$OLD" --variant LX_ROLLOUT_MINB=4 >> gpurun_out/ab_r2v.jsonl 2>>gpurun_out/ab_r2v.err
timeout 300 python tools/ab_env.py --game pente --reps 6 --variant "" --variant "$OLD" --variant LX_ROLLOUT_MINB=5 >> gpurun_out/ab_r2v.jsonl 2>>gpurun_out/ab_r2v.err
python - <<'PY'
import json
for line in open("gpurun_out/ab_r2v.jsonl"):
    d = json.loads(line)
    print(d["game"], d["same_stats"], [(v["env"], round(v["env_steps_per_s"] / 1e9, 2)) for v in d["variants"]])
PY
