# r1n: rollout block-occupancy A/B per config game (same seeds, stats compared):
# 2 x 256 (default) vs 3 x 256 / 4 x 256 / 6 x 128 resident blocks per SM.
mkdir -p gpurun_out
for g in connect_four tic_tac_toe hex reversi pente; do
  timeout 400 python tools/ab_env.py --game $g --variant "" --variant LX_ROLLOUT_MINB=3 \
      --variant LX_ROLLOUT_MINB=4 --variant LX_ROLLOUT_THREADS=128,LX_ROLLOUT_MINB=6 \
      > gpurun_out/ab_minb_$g.json 2>&1
  python -c "
import json,sys
d=json.load(open('gpurun_out/ab_minb_$g.json'))
print(d['game'], d['same_stats'], [(v['env'], round(v['env_steps_per_s']/1e9,2)) for v in d['variants']])
" || tail -3 gpurun_out/ab_minb_$g.json
done
