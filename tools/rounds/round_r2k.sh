# r2k: register cap of the per-ply kernels (LX_STEP_MINB) A/B
mkdir -p gpurun_out
rm -f gpurun_out/ab_r2k.jsonl
for g in connect_four tic_tac_toe hex reversi pente; do
  timeout 900 python tools/ab_envstep.py --game $g --variant "" --variant LX_STEP_MINB=4 --variant LX_STEP_MINB=6 >> gpurun_out/ab_r2k.jsonl 2>> gpurun_out/ab_r2k.err
  echo "$g rc=$?"
done
python - <<'PY'
import json
for line in open("gpurun_out/ab_r2k.jsonl"):
    d = json.loads(line)
    print(d["game"], [(v["env"], round(v["random_step_G"], 1), round(v["env_bool_G"], 1), round(v["env_bits_G"], 1)) for v in d["variants"]])
PY
timeout 600 python tools/ab_env.py --game tic_tac_toe --reps 10 --variant "" --variant LX_PLY_UNROLL=4 > gpurun_out/ab_r2k_unroll.jsonl 2>> gpurun_out/ab_r2k.err
timeout 600 python tools/ab_env.py --game reversi --reps 10 --variant "" --variant LX_PLY_UNROLL=3 >> gpurun_out/ab_r2k_unroll.jsonl 2>> gpurun_out/ab_r2k.err
python - <<'PY'
import json
for line in open("gpurun_out/ab_r2k_unroll.jsonl"):
    d = json.loads(line)
    print(d["game"], d["same_stats"], [(v["env"], round(v["env_steps_per_s"] / 1e9, 2)) for v in d["variants"]])
PY
