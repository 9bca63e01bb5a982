mkdir -p gpurun_out
for g in connect_four tic_tac_toe; do
  timeout 900 python tools/e2e_sweep.py --game $g --min-log2 10 --max-log2 22 >> gpurun_out/e2e_sweep.jsonl 2>> gpurun_out/e2e_sweep.err
done
python - <<'PY'
import json
for l in open("gpurun_out/e2e_sweep.jsonl"):
    d = json.loads(l)
    print(d["game"], d["batch"], round(d["e2e_env_steps_per_s"] / 1e9, 3), round(d["device_env_steps_per_s"] / 1e9, 3), round(d["us_per_episode_e2e"], 1))
PY
tail -3 gpurun_out/e2e_sweep.err
