# zero-copy small-batch lx_playout_host
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_playout_host.py tests/test_c_abi.py -m gpu -q -x > gpurun_out/pytest_zc.log 2>&1; tail -3 gpurun_out/pytest_zc.log
timeout 300 python tools/probe_playout_host.py --game tic_tac_toe --batch 1024 --reps 300 2>&1 | tail -1
timeout 300 python tools/probe_playout_host.py --game tic_tac_toe --batch 8192 --reps 300 2>&1 | tail -1
timeout 300 python tools/probe_playout_host.py --game connect_four --batch 1024 --reps 300 2>&1 | tail -1
