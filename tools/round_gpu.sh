mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -8 gpurun_out/smoke.log
python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; tail -c 3000 gpurun_out/bench_c4.json
python bench.py --impl reference --steps 20 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; tail -c 1500 gpurun_out/bench_ref.json
python bench.py --game english_draughts --steps 20 > gpurun_out/bench_draughts.json 2>&1
python bench.py --steps 3 --warmup 1 --no-extras > gpurun_out/b_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 1 --no-extras > gpurun_out/ncu_launch.log 2>&1; echo "launches rc=$?"
NO_LAUNCHES=1 GAMES="connect_four:4194304 tic_tac_toe:4194304 hex:4194304 reversi:4194304 pente:4194304 gomoku:4194304 yavalath:4194304 english_draughts:4194304 dai_hasami_shogi:4194304 wolf_and_sheep:4194304 gridworld:4194304" bash tools/profile_all.sh
python tools/mcts_bench.py --game connect_four --games 16 > gpurun_out/mcts_c4.json 2>&1
python tools/mcts_bench.py --gavel --game connect_four --matches 24 > gpurun_out/gavel_c4.json 2>&1
python tools/mcts_bench.py --game reversi --games 8 --strong 50 --weak 25 > gpurun_out/mcts_rev.json 2>&1
python tools/mcts_bench.py --game tic_tac_toe --games 32 > gpurun_out/mcts_ttt.json 2>&1
cat gpurun_out/mcts_*.json
