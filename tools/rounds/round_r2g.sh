# r2g: A/B of rollout ply changes: mirrored capture block + stashed word
# select (Pente / Gomoku), funnel shifts as IMAD pairs on the FMA pipe (all)
mkdir -p gpurun_out
rm -f gpurun_out/ab_r2g.jsonl
for g in pente gomoku; do
  timeout 900 python tools/ab_env.py --game $g --reps 6 --variant LX_CAPTURE_FAST=0,LX_SELECT_STASH=0 \
      --variant LX_SELECT_STASH=0 --variant LX_CAPTURE_FAST=0 --variant "" --variant LX_SHIFT_FMA=1 >> gpurun_out/ab_r2g.jsonl 2>> gpurun_out/ab_r2g.err
  echo "$g rc=$?"
done
for g in connect_four tic_tac_toe hex reversi yavalath; do
  timeout 900 python tools/ab_env.py --game $g --reps 10 --variant "" --variant LX_SHIFT_FMA=1 >> gpurun_out/ab_r2g.jsonl 2>> gpurun_out/ab_r2g.err
  echo "$g rc=$?"
done
python - <<'PY'
import json
for line in open("gpurun_out/ab_r2g.jsonl"):
    d = json.loads(line)
    print(d["game"], d["same_stats"], [(v["env"], round(v["env_steps_per_s"] / 1e9, 2)) for v in d["variants"]])
PY
