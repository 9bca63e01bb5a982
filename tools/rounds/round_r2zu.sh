# ncu of one lx_mcts launch (C4 16-game match, MCTS-100 vs -50): lanes, issue, stalls
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none -k regex:"^lx_mcts\$" -s 40 -c 1 -o gpurun_out/mcts_c4 \
   python tools/mcts_bench.py --game connect_four --games 16 --no-reference > gpurun_out/ncu_mcts.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/mcts_c4.ncu-rep --page details --csv > gpurun_out/mcts_c4_details.csv 2>/dev/null
ncu -i gpurun_out/mcts_c4.ncu-rep --page raw --csv --metrics smsp__thread_inst_executed_per_inst_executed.ratio,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum,launch__grid_size,launch__block_size,smsp__average_warp_latency_issue_stalled_wait,smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio > gpurun_out/mcts_c4_raw.csv 2>/dev/null
rm -f gpurun_out/*.ncu-rep
head -5 gpurun_out/mcts_c4_raw.csv | cut -c1-600
