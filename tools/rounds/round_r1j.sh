mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -8 gpurun_out/smoke.log
python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; tail -c 3000 gpurun_out/bench_c4.json
python bench.py --impl reference --steps 20 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; tail -c 1500 gpurun_out/bench_ref.json
NO_LAUNCHES= GAMES="connect_four:4194304" bash tools/profile_all.sh
LX_FUZZ_ALL=2/4 timeout 1500 python -m pytest tests/test_fuzz_corpus.py -m gpu -q -k "device" > gpurun_out/fuzz_2of4.log 2>&1; tail -2 gpurun_out/fuzz_2of4.log
