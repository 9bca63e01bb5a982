# r2n: Kogge-Stone pre-masked propagator A/B (Reversi), agents after the meta/counts fusion
mkdir -p gpurun_out
timeout 600 python tools/ab_env.py --game reversi --reps 10 --variant LX_KS_PREMASK=0 --variant "" > gpurun_out/ab_r2n.jsonl 2> gpurun_out/ab_r2n.err
timeout 600 python tools/ab_envstep.py --game reversi --variant LX_KS_PREMASK=0 --variant "" >> gpurun_out/ab_r2n.jsonl 2>> gpurun_out/ab_r2n.err
tail -c 600 gpurun_out/ab_r2n.jsonl
timeout 900 python -m pytest tests/test_gpu_agents.py tests/test_gpu_device_binding.py -q -x > gpurun_out/pytest_agents.log 2>&1; tail -2 gpurun_out/pytest_agents.log
timeout 600 python tools/mcts_bench.py --game connect_four --games 16 > gpurun_out/mcts_c4.json 2>&1; tail -c 400 gpurun_out/mcts_c4.json
timeout 600 python tools/mcts_bench.py --game tic_tac_toe --games 32 > gpurun_out/mcts_ttt.json 2>&1; tail -c 400 gpurun_out/mcts_ttt.json
timeout 600 python tools/mcts_bench.py --gavel --game connect_four --matches 24 > gpurun_out/gavel_c4.json 2>&1; tail -c 400 gpurun_out/gavel_c4.json
