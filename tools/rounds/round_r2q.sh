# r2q: bit masks stored per lane as one vector store; TTT refill 12/8
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_env.py -q -x > gpurun_out/pytest_env.log 2>&1; tail -2 gpurun_out/pytest_env.log
rm -f gpurun_out/ab_r2q.jsonl
for g in connect_four tic_tac_toe hex reversi; do
  timeout 600 python tools/ab_envstep.py --game $g --variant "" >> gpurun_out/ab_r2q.jsonl 2>> gpurun_out/ab_r2q.err
done
python - <<'PY'
import json
for line in open("gpurun_out/ab_r2q.jsonl"):
    d = json.loads(line)
    print(d["game"], [(v["env"], round(v["random_step_G"], 1), round(v["env_bool_G"], 1), round(v["env_bits_G"], 1)) for v in d["variants"]])
PY
timeout 600 python tools/ab_env.py --game tic_tac_toe --reps 10 --variant "" --variant LX_REFILL_LANES=16,LX_REFILL_WAIT=12 --variant LX_REFILL_LANES=12,LX_REFILL_WAIT=12 > gpurun_out/ab_r2q_ttt.jsonl 2>> gpurun_out/ab_r2q.err
python - <<'PY'
import json
for line in open("gpurun_out/ab_r2q_ttt.jsonl"):
    d = json.loads(line)
    print(d["game"], d["same_stats"], [(v["env"], round(v["env_steps_per_s"] / 1e9, 2)) for v in d["variants"]])
PY
