# every-env parity of full 2^22 episodes for the three games bench samples at 2^20
mkdir -p gpurun_out
timeout 1500 python tools/full_parity.py --games hex,reversi,pente > gpurun_out/full_parity.jsonl 2> gpurun_out/full_parity.err; echo "rc=$?"
python - <<'PY'
import json
for line in open("gpurun_out/full_parity.jsonl"):
    d = json.loads(line)
    print(d["game"], d["parity"]["envs_checked"], d["parity"]["mismatches"], round(d["oracle"]["value"] / 1e6, 2), "M/s oracle", d["oracle"]["sample"][-40:])
PY
tail -3 gpurun_out/full_parity.err
