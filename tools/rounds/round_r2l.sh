# r2l: full check of the current build: GPU suite, smoke, ncu of the five config
# games (rollout + per-ply kernels), sweep; the bench runs after the profiles
# are summarised and committed (next call), so its roofline reads fresh counts.
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -4 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -3 gpurun_out/smoke.log
NO_LAUNCHES=1 STEP_GAMES="connect_four:4194304 tic_tac_toe:4194304 hex:4194304 reversi:4194304 pente:4194304" bash tools/profile_all.sh
timeout 900 python tools/sweep.py --min-log2 10 --max-log2 22 > gpurun_out/sweep.jsonl 2> gpurun_out/sweep.err; echo "sweep rc=$?"
for g in connect_four hex; do
  timeout 600 ncu --set full --clock-control none -k regex:"lx_export|lx_observe" -s 2 -c 2 -o gpurun_out/exportprof_$g python tools/ncu_export.py --game $g > gpurun_out/ncu_export_$g.log 2>&1; echo "$g export rc=$?"
done
