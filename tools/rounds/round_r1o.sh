# r1o: occupancy A/B for the six non-config corpus games + PGX env path timing fix check.
mkdir -p gpurun_out
for g in gomoku yavalath english_draughts dai_hasami_shogi wolf_and_sheep gridworld; do
  timeout 400 python tools/ab_env.py --game $g --variant "" --variant LX_ROLLOUT_MINB=3 \
      --variant LX_ROLLOUT_MINB=4 > gpurun_out/ab_minb_$g.json 2>&1
  python -c "
import json
d=json.load(open('gpurun_out/ab_minb_$g.json'))
print(d['game'], d['same_stats'], [(v['env'], round(v['env_steps_per_s']/1e9,2)) for v in d['variants']])
" || tail -3 gpurun_out/ab_minb_$g.json
done
timeout 300 python tools/env_bench.py --batch 4194304 > gpurun_out/env_bench.jsonl 2>&1; cat gpurun_out/env_bench.jsonl
