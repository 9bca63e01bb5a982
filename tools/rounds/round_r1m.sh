# r1m: round-end refresh on the current build (Hex cooperative flood + Pente
# mirror captures): GPU suite, smoke, fresh ncu of the five config games and
# summaries written on the box (so bench.py reads a current profile), bench
# C4 + reference arm, launch list.
mkdir -p gpurun_out/profiles
python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -8 gpurun_out/smoke.log
GAMES="connect_four:4194304 tic_tac_toe:4194304 hex:4194304 reversi:4194304 pente:4194304" bash tools/profile_all.sh
python tools/ncu_summary.py gpurun_out --tag ${TAG:-r1m} > gpurun_out/summary.log 2>&1; cat gpurun_out/summary.log
cp profiles/${TAG:-r1m}_* profiles/rollout_*.json gpurun_out/profiles/
python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; tail -c 3000 gpurun_out/bench_c4.json
python bench.py --impl reference --steps 20 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; tail -c 1500 gpurun_out/bench_ref.json
for g in hex reversi pente tic_tac_toe; do
  python bench.py --game $g --steps 50 --no-extras > gpurun_out/bench_$g.json 2>&1; tail -c 700 gpurun_out/bench_$g.json; echo
done
for g in yavalath wolf_and_sheep english_draughts gridworld; do
  python bench.py --game $g --steps 50 --no-extras > gpurun_out/bench_$g.json 2>&1; tail -c 300 gpurun_out/bench_$g.json; echo
done
