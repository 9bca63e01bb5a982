# r2m: full check after the export alignment fix; profiles summarised on the box
# so the bench in this call reads this build's counts; sweep; reference arm.
mkdir -p gpurun_out/profiles_r2m
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -4 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -3 gpurun_out/smoke.log
NO_LAUNCHES=1 STEP_GAMES="connect_four:4194304 tic_tac_toe:4194304 hex:4194304 reversi:4194304 pente:4194304" bash tools/profile_all.sh
python tools/ncu_summary.py gpurun_out --tag r2m --out profiles > gpurun_out/ncu_summary.log 2>&1; tail -6 gpurun_out/ncu_summary.log
cp profiles/rollout_*.json profiles/step_*.json profiles/r2m_* gpurun_out/profiles_r2m/ 2>/dev/null
for g in connect_four hex; do
  timeout 600 ncu --set full --clock-control none -k regex:"lx_export|lx_observe" -s 2 -c 2 -o gpurun_out/exportprof_$g python tools/ncu_export.py --game $g > gpurun_out/ncu_export_$g.log 2>&1; echo "$g export rc=$?"
done
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench rc=$?"; tail -c 300 gpurun_out/bench_c4.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout 300 python bench.py --steps 3 --warmup 1 --no-extras > gpurun_out/b_plain.log 2>&1 && timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 1 --no-extras > gpurun_out/ncu_launch.log 2>&1; echo "launches rc=$?"
timeout 900 python tools/sweep.py --min-log2 10 --max-log2 22 > gpurun_out/sweep.jsonl 2> gpurun_out/sweep.err; echo "sweep rc=$?"
