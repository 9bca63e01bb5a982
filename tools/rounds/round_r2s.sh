mkdir -p gpurun_out
timeout 900 python tools/ab_env.py --game hex --reps 10 --variant LX_SPLIT_FLOOD=0 --variant LX_ROLLOUT_MINB=2 \
   --variant LX_ROLLOUT_MINB=2,LX_SPLIT_FLOOD=0 --variant LX_ROLLOUT_MINB=2,LX_PLY_UNROLL=1 > gpurun_out/ab_r2s.jsonl 2> gpurun_out/ab_r2s.err
python - <<'PY'
import json
for line in open("gpurun_out/ab_r2s.jsonl"):
    d = json.loads(line)
    print(d["game"], d["same_stats"], [(v["env"], round(v["env_steps_per_s"] / 1e9, 2)) for v in d["variants"]])
PY
