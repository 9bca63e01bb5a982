mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_playout_host.py -m gpu -q > gpurun_out/pytest_ph.log 2>&1; tail -15 gpurun_out/pytest_ph.log
