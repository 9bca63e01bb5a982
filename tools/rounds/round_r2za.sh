# bool-mask writer from one concatenated bit stream: tests + env-step A/B
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_env.py tests/test_gpu_parity.py tests/test_gpu_mover.py tests/test_gpu_movement.py -m gpu -q -x > gpurun_out/pytest_mask.log 2>&1; tail -3 gpurun_out/pytest_mask.log
for g in connect_four tic_tac_toe hex reversi pente; do
  timeout 300 python tools/ab_envstep.py --game $g --variant "" --variant LX_MASK_STREAM=0 >> gpurun_out/ab_r2za.jsonl 2>>gpurun_out/ab_r2za.err
done
python - <<'PY'
import json
for line in open("gpurun_out/ab_r2za.jsonl"):
    d = json.loads(line)
    print(d["game"], [(v["env"], round(v["env_bool_G"], 2), round(v["env_bits_G"], 2), v.get("mask_sum_bool"), v.get("mask_sum_bits")) for v in d["variants"]])
PY
