# final check of a build: GPU suite, smoke, ncu of the five config games
# (rollout + per-ply kernels) summarised on the box so the bench in this call
# reads this build's counts, bench (both arms), sweep, launch list.  Reports
# are deleted after summarising (gpurun merges <= 64 MiB back).
TAG=${TAG:-r2final}
mkdir -p gpurun_out/profiles_$TAG
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -4 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -3 gpurun_out/smoke.log
NO_LAUNCHES=1 STEP_GAMES="connect_four:4194304 tic_tac_toe:4194304 hex:4194304 reversi:4194304 pente:4194304" bash tools/profile_all.sh > gpurun_out/profile_all.log 2>&1
python tools/ncu_summary.py gpurun_out --tag $TAG --out profiles > gpurun_out/ncu_summary.log 2>&1; tail -6 gpurun_out/ncu_summary.log
cp profiles/rollout_*.json profiles/step_*.json profiles/${TAG}_* gpurun_out/profiles_$TAG/ 2>/dev/null
for g in connect_four hex; do
  timeout 600 ncu --set full --clock-control none -k regex:"lx_export|lx_observe" -s 2 -c 2 -o gpurun_out/exportprof_$g python tools/ncu_export.py --game $g > gpurun_out/ncu_export_$g.log 2>&1; echo "$g export rc=$?"
  ncu -i gpurun_out/exportprof_$g.ncu-rep --page raw --csv > gpurun_out/profiles_$TAG/export_raw_$g.csv 2>/dev/null
done
mkdir -p gpurun_out/sass_keep && cp gpurun_out/sass_connect_four.csv gpurun_out/sass_pente.csv gpurun_out/sass_keep/ 2>/dev/null
rm -f gpurun_out/*.ncu-rep gpurun_out/sass_*.csv
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench rc=$?"; tail -c 300 gpurun_out/bench_c4.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout 300 python bench.py --steps 3 --warmup 1 --no-extras > gpurun_out/b_plain.log 2>&1 && timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 1 --no-extras > gpurun_out/ncu_launch.log 2>&1; echo "launches rc=$?"
timeout 900 python tools/sweep.py --min-log2 10 --max-log2 22 > gpurun_out/sweep.jsonl 2> gpurun_out/sweep.err; echo "sweep rc=$?"
du -sh gpurun_out
timeout 600 python tools/mcts_bench.py --game connect_four --games 16 > gpurun_out/mcts_c4.json 2>&1; tail -c 300 gpurun_out/mcts_c4.json
timeout 600 python tools/mcts_bench.py --game reversi --games 8 --strong 50 --weak 25 > gpurun_out/mcts_rev.json 2>&1; tail -c 300 gpurun_out/mcts_rev.json
timeout 600 python tools/mcts_bench.py --gavel --game connect_four --matches 24 > gpurun_out/gavel_c4.json 2>&1; tail -c 300 gpurun_out/gavel_c4.json
# small-batch latency and the host-buffer C-ABI call on this build
timeout 300 python tools/latency_probe.py --game tic_tac_toe --batch 1024 --caps 0,9,200 > gpurun_out/profiles_$TAG/lat_ttt1024.jsonl 2>&1
timeout 300 python tools/probe_playout_host.py > gpurun_out/profiles_$TAG/playout_host_c4.jsonl 2>&1
timeout 300 python tools/probe_playout_host.py --game tic_tac_toe --batch 1024 --reps 300 >> gpurun_out/profiles_$TAG/playout_host_c4.jsonl 2>&1
cp gpurun_out/bench_c4.json gpurun_out/profiles_$TAG/bench.json; cp gpurun_out/bench_ref.json gpurun_out/profiles_$TAG/bench_reference.json
cp gpurun_out/sweep.jsonl gpurun_out/launches.csv gpurun_out/pytest_gpu.log gpurun_out/smoke.log gpurun_out/mcts_c4.json gpurun_out/mcts_rev.json gpurun_out/gavel_c4.json gpurun_out/profiles_$TAG/ 2>/dev/null
du -sh gpurun_out
