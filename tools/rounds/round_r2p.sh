# r2p: refill thresholds re-tuned with multi-ply passes (LX_REFILL_LANES / WAIT)
mkdir -p gpurun_out
rm -f gpurun_out/ab_r2p.jsonl
timeout 900 python tools/ab_env.py --game connect_four --reps 10 --variant "" --variant LX_REFILL_LANES=4,LX_REFILL_WAIT=4 \
   --variant LX_REFILL_LANES=3,LX_REFILL_WAIT=2 --variant LX_REFILL_LANES=8,LX_REFILL_WAIT=6 --variant LX_REFILL_LANES=2,LX_REFILL_WAIT=1 >> gpurun_out/ab_r2p.jsonl 2>> gpurun_out/ab_r2p.err
timeout 900 python tools/ab_env.py --game tic_tac_toe --reps 10 --variant "" --variant LX_REFILL_LANES=6,LX_REFILL_WAIT=4 \
   --variant LX_REFILL_LANES=4,LX_REFILL_WAIT=2 --variant LX_REFILL_LANES=12,LX_REFILL_WAIT=8 >> gpurun_out/ab_r2p.jsonl 2>> gpurun_out/ab_r2p.err
timeout 900 python tools/ab_env.py --game hex --reps 6 --variant "" --variant LX_REFILL_LANES=2,LX_REFILL_WAIT=2 \
   --variant LX_REFILL_LANES=4,LX_REFILL_WAIT=4 >> gpurun_out/ab_r2p.jsonl 2>> gpurun_out/ab_r2p.err
timeout 900 python tools/ab_env.py --game reversi --reps 6 --variant "" --variant LX_REFILL_LANES=2,LX_REFILL_WAIT=2 \
   --variant LX_REFILL_LANES=4,LX_REFILL_WAIT=4 >> gpurun_out/ab_r2p.jsonl 2>> gpurun_out/ab_r2p.err
python - <<'PY'
import json
for line in open("gpurun_out/ab_r2p.jsonl"):
    d = json.loads(line)
    print(d["game"], d["same_stats"], [(v["env"], round(v["env_steps_per_s"] / 1e9, 2)) for v in d["variants"]])
PY
