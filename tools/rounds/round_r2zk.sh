# early draw (RNG chain ahead of the legality): tests + latency + throughput + MCTS A/B
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_agents.py -m gpu -q -x > gpurun_out/pytest_early.log 2>&1; tail -2 gpurun_out/pytest_early.log
for g in tic_tac_toe connect_four; do
  for v in "" "LX_EARLY_DRAW=0"; do
    timeout 300 python tools/latency_probe.py --game $g --batch 1024 --caps 200 --variant "$v" 2>&1 | grep -v trivial
  done
done | tee gpurun_out/lat_early.jsonl
for g in connect_four tic_tac_toe hex reversi pente; do
  timeout 300 python tools/ab_env.py --game $g --reps 8 --variant "" --variant LX_EARLY_DRAW=0 >> gpurun_out/ab_r2zk.jsonl 2>>gpurun_out/ab_r2zk.err
done
python - <<'PY'
import json
for line in open("gpurun_out/ab_r2zk.jsonl"):
    d = json.loads(line)
    print(d["game"], d["same_stats"], [(v["env"], round(v["env_steps_per_s"] / 1e9, 2)) for v in d["variants"]])
PY
timeout 600 python tools/mcts_bench.py --game connect_four --games 16 --no-reference > gpurun_out/mcts_early1.json 2>&1 || timeout 600 python tools/mcts_bench.py --game connect_four --games 16 > gpurun_out/mcts_early1.json 2>&1; tail -c 250 gpurun_out/mcts_early1.json; echo
LX_EARLY_DRAW=0 timeout 600 python tools/mcts_bench.py --game connect_four --games 16 --no-reference > gpurun_out/mcts_early0.json 2>&1 || LX_EARLY_DRAW=0 timeout 600 python tools/mcts_bench.py --game connect_four --games 16 > gpurun_out/mcts_early0.json 2>&1; tail -c 250 gpurun_out/mcts_early0.json
