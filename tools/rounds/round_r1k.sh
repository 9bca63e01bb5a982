# r1k: cooperative reach-set flood -- GPU suite, A/B vs the per-lane flood,
# ncu of Hex + C4, summaries written on the box so bench.py reads fresh ones.
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
python tools/ab_flood.py --game hex > gpurun_out/ab_flood_hex.json 2>&1; cat gpurun_out/ab_flood_hex.json
NO_LAUNCHES=1 GAMES="hex:4194304 connect_four:4194304" bash tools/profile_all.sh
python tools/ncu_summary.py gpurun_out --tag r1k > gpurun_out/summary.log 2>&1; cat gpurun_out/summary.log
mkdir -p gpurun_out/profiles && cp profiles/r1k_* profiles/rollout_Hex.json profiles/rollout_Connect_Four.json gpurun_out/profiles/
python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; tail -c 1500 gpurun_out/bench_c4.json
python bench.py --game hex --steps 50 --no-extras > gpurun_out/bench_hex.json 2>&1; tail -c 600 gpurun_out/bench_hex.json
