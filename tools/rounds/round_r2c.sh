# r2c: full GPU suite (no -x: list every failure) incl. mover fixtures, C caller,
# reference loops/tests over the adapter.
mkdir -p gpurun_out
timeout 2000 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -15 gpurun_out/pytest_gpu.log
tail -30 gpurun_out/ref_tests_over_adapter.log
