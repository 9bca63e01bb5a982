# knob re-check on the current build (2^22, same stats required)
mkdir -p gpurun_out
timeout 400 python tools/ab_env.py --game hex --reps 8 --variant "" --variant LX_ROLLOUT_MINB=4 --variant LX_PLY_UNROLL=1 --variant LX_REFILL_LANES=4,LX_REFILL_WAIT=4 >> gpurun_out/ab_r2zb.jsonl 2>>gpurun_out/ab_r2zb.err
timeout 400 python tools/ab_env.py --game tic_tac_toe --reps 10 --variant "" --variant LX_ROLLOUT_MINB=5 --variant LX_REFILL_LANES=20,LX_REFILL_WAIT=16 --variant LX_ROLLOUT_THREADS=128,LX_ROLLOUT_MINB=8 >> gpurun_out/ab_r2zb.jsonl 2>>gpurun_out/ab_r2zb.err
timeout 400 python tools/ab_env.py --game reversi --reps 8 --variant "" --variant LX_SHIFT_FMA=0 --variant LX_PLY_UNROLL=2 --variant LX_ROLLOUT_THREADS=128,LX_ROLLOUT_MINB=6 >> gpurun_out/ab_r2zb.jsonl 2>>gpurun_out/ab_r2zb.err
timeout 400 python tools/ab_env.py --game connect_four --reps 10 --variant "" --variant LX_ROLLOUT_THREADS=128,LX_ROLLOUT_MINB=8 --variant LX_REFILL_LANES=8,LX_REFILL_WAIT=8 --variant LX_PLY_UNROLL=4 >> gpurun_out/ab_r2zb.jsonl 2>>gpurun_out/ab_r2zb.err
timeout 400 python tools/ab_env.py --game pente --reps 5 --variant "" --variant LX_ROLLOUT_MINB=5 --variant LX_PLY_UNROLL=2 >> gpurun_out/ab_r2zb.jsonl 2>>gpurun_out/ab_r2zb.err
python - <<'PY'
import json
for line in open("gpurun_out/ab_r2zb.jsonl"):
    d = json.loads(line)
    print(d["game"], d["same_stats"], [(v["env"], round(v["env_steps_per_s"] / 1e9, 2)) for v in d["variants"]])
PY
