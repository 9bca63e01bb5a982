# r2e: A/B of the rollout variants (SWAR select, 2 plies per refill pass)
mkdir -p gpurun_out
for g in connect_four tic_tac_toe hex reversi pente; do
  timeout 600 python tools/ab_env.py --game $g --reps 10 --variant LX_SELECT_SWAR=0 --variant "" \
      --variant LX_PLY_UNROLL=2 --variant LX_PLY_UNROLL=2,LX_SELECT_SWAR=0 >> gpurun_out/ab_r2e.jsonl 2>> gpurun_out/ab_r2e.err
  echo "$g rc=$?"
done
python - <<'PY'
import json
for line in open("gpurun_out/ab_r2e.jsonl"):
    d = json.loads(line)
    print(d["game"], d["same_stats"], [(v["env"], round(v["env_steps_per_s"] / 1e9, 2)) for v in d["variants"]])
PY
# warp-per-tree device MCTS (shared-memory trees): tests vs host search / reference, match timing
timeout 900 python -m pytest tests/test_gpu_agents.py -q -x > gpurun_out/pytest_agents.log 2>&1; tail -3 gpurun_out/pytest_agents.log
timeout 600 python tools/mcts_bench.py --game connect_four --games 16 > gpurun_out/mcts_c4.json 2>&1; tail -c 600 gpurun_out/mcts_c4.json
timeout 600 python tools/mcts_bench.py --game reversi --games 8 --strong 50 --weak 25 > gpurun_out/mcts_rev.json 2>&1; tail -c 600 gpurun_out/mcts_rev.json
timeout 600 python tools/mcts_bench.py --game tic_tac_toe --games 32 > gpurun_out/mcts_ttt.json 2>&1; tail -c 600 gpurun_out/mcts_ttt.json
