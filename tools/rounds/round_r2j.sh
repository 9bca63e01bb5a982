# r2j: int lane flags in lx_rollout; unroll-3 A/B; ncu of the interchange kernels
mkdir -p gpurun_out
timeout 600 python tools/ab_env.py --game connect_four --reps 10 --variant "" --variant LX_PLY_UNROLL=3 > gpurun_out/ab_r2j.jsonl 2> gpurun_out/ab_r2j.err
timeout 600 python tools/ab_env.py --game tic_tac_toe --reps 10 --variant "" --variant LX_PLY_UNROLL=3 >> gpurun_out/ab_r2j.jsonl 2>> gpurun_out/ab_r2j.err
timeout 600 python tools/ab_env.py --game hex --reps 10 --variant "" --variant LX_PLY_UNROLL=1 >> gpurun_out/ab_r2j.jsonl 2>> gpurun_out/ab_r2j.err
python - <<'PY'
import json
for line in open("gpurun_out/ab_r2j.jsonl"):
    d = json.loads(line)
    print(d["game"], d["same_stats"], [(v["env"], round(v["env_steps_per_s"] / 1e9, 2)) for v in d["variants"]])
PY
for g in connect_four hex; do
  timeout 300 python tools/ncu_export.py --game $g > gpurun_out/export_$g.txt 2>&1 && \
  timeout 600 ncu --set full --clock-control none -k regex:"lx_export|lx_observe" -s 2 -c 2 -o gpurun_out/exportprof_$g python tools/ncu_export.py --game $g > gpurun_out/ncu_export_$g.log 2>&1; echo "$g export rc=$?"
done
