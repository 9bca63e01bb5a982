mkdir -p gpurun_out
timeout 300 python tools/probe_playout_host.py > gpurun_out/probe_ph.jsonl 2>&1; cat gpurun_out/probe_ph.jsonl
timeout 300 python tools/probe_playout_host.py --game tic_tac_toe --batch 1024 --reps 200 >> gpurun_out/probe_ph.jsonl 2>&1; tail -1 gpurun_out/probe_ph.jsonl
for g in pente hex connect_four; do
  timeout 300 python tools/ab_env.py --game $g --reps 8 --variant "" --variant LX_SEED_STREAM=0 --variant "" >> gpurun_out/ab_r2x.jsonl 2>>gpurun_out/ab_r2x.err
done
python - <<'PY'
import json
for line in open("gpurun_out/ab_r2x.jsonl"):
    d = json.loads(line)
    print(d["game"], d["same_stats"], [(v["env"], round(v["env_steps_per_s"] / 1e9, 2)) for v in d["variants"]])
PY
