mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_playout_host.py tests/test_c_abi.py -m gpu -q > gpurun_out/pytest_ph.log 2>&1; tail -3 gpurun_out/pytest_ph.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench rc=$?"; tail -c 300 gpurun_out/bench_c4.err
python tools/bench_table.py gpurun_out/bench_c4.json
