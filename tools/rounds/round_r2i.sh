# r2i: Hex neighbour table A/B; MCTS host-side trims + launch list of the C4 match
mkdir -p gpurun_out
timeout 600 python tools/ab_env.py --game hex --reps 10 --variant LX_NEIGHBOR_TABLE=0 --variant "" > gpurun_out/ab_r2i.jsonl 2> gpurun_out/ab_r2i.err
timeout 600 python tools/ab_env.py --game yavalath --reps 10 --variant LX_NEIGHBOR_TABLE=0 --variant "" >> gpurun_out/ab_r2i.jsonl 2>> gpurun_out/ab_r2i.err
python - <<'PY'
import json
for line in open("gpurun_out/ab_r2i.jsonl"):
    d = json.loads(line)
    print(d["game"], d["same_stats"], [(v["env"], round(v["env_steps_per_s"] / 1e9, 2)) for v in d["variants"]])
PY
timeout 900 python -m pytest tests/test_gpu_agents.py -q -x > gpurun_out/pytest_agents.log 2>&1; tail -2 gpurun_out/pytest_agents.log
timeout 600 python tools/mcts_bench.py --game connect_four --games 16 > gpurun_out/mcts_c4.json 2>&1; tail -c 400 gpurun_out/mcts_c4.json
timeout 600 python tools/mcts_bench.py --game reversi --games 8 --strong 50 --weak 25 > gpurun_out/mcts_rev.json 2>&1; tail -c 400 gpurun_out/mcts_rev.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/mcts_launches.csv python tools/mcts_bench.py --game connect_four --games 16 --no-reference > gpurun_out/mcts_ncu.log 2>&1; echo "ncu rc=$?"
python - <<'PY'
import csv, collections
rows = [r for r in csv.reader(open("gpurun_out/mcts_launches.csv")) if len(r) > 5]
h = rows[0]; ik = h.index("Kernel Name"); iv = h.index("Metric Value")
c = collections.defaultdict(list)
for r in rows[1:]:
    try: c[r[ik][:40]].append(float(r[iv].replace(",", "")))
    except ValueError: pass
for k, v in sorted(c.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k:40s} n={len(v):5d} total={sum(v)/1e6:8.2f} ms mean={sum(v)/len(v)/1e3:8.1f} us")
PY
