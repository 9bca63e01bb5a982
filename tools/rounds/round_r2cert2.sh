# certification of the final tree: full GPU suite, smoke, bench (both arms), MCTS
mkdir -p gpurun_out/final_cert2
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/final_cert2/pytest_gpu.log 2>&1; tail -3 gpurun_out/final_cert2/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_cert2/smoke.log 2>&1; tail -2 gpurun_out/final_cert2/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/final_cert2/bench.json 2> gpurun_out/final_cert2/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/final_cert2/bench_reference.json 2> gpurun_out/final_cert2/bench_reference.err; echo "ref rc=$?"
python tools/bench_table.py gpurun_out/final_cert2/bench.json
timeout 600 python tools/mcts_bench.py --game connect_four --games 16 > gpurun_out/final_cert2/mcts_c4.json 2>&1; tail -c 300 gpurun_out/final_cert2/mcts_c4.json
