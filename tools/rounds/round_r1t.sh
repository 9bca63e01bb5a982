# r1t: device MCTS kernel (lx_mcts) profile + final GPU suite on the committed tree.
mkdir -p gpurun_out
python tools/mcts_bench.py --no-reference --games 16 > gpurun_out/mcts_plain.log 2>&1; tail -3 gpurun_out/mcts_plain.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/mcts_launches.csv \
    python tools/mcts_bench.py --no-reference --games 16 > gpurun_out/mcts_ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:lx_mcts -s 3 -c 1 -f -o gpurun_out/mcts_c4 \
    python tools/mcts_bench.py --no-reference --games 16 > gpurun_out/mcts_ncu2.log 2>&1; tail -2 gpurun_out/mcts_ncu2.log
python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -3 gpurun_out/smoke.log
