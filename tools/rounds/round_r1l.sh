# r1l: Pente captures through the mirror, block-occupancy A/B per game.
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
for g in connect_four tic_tac_toe yavalath wolf_and_sheep gridworld; do
  timeout 300 python tools/ab_env.py --game $g --variant LX_ROLLOUT_MINB=2 --variant LX_ROLLOUT_MINB=3 --variant LX_ROLLOUT_MINB=4 > gpurun_out/ab_minb_$g.json 2>&1; cut -c1-600 gpurun_out/ab_minb_$g.json
done
for g in pente hex reversi gomoku english_draughts; do
  timeout 300 python tools/ab_env.py --game $g --variant LX_ROLLOUT_MINB=2 --variant LX_ROLLOUT_MINB=3 > gpurun_out/ab_minb_$g.json 2>&1; cut -c1-600 gpurun_out/ab_minb_$g.json
done
