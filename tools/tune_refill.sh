#!/bin/bash
# GPU box: sweep the batched game-over thresholds (LX_REFILL_LANES/WAIT)
mkdir -p gpurun_out
for kw in ${KW:-1:1 4:4 6:6 8:8 12:12}; do
  k=${kw%%:*}; w=${kw##*:}
  LX_REFILL_LANES=$k LX_REFILL_WAIT=$w timeout 300 python tools/sweep.py --min-log2 22 --seconds 0.4 \
     --games ${GAMES:-tic_tac_toe,connect_four,hex,reversi,pente} | sed "s/^/{\"K\":$k,\"T\":$w,\"r\":/; s/$/}/"
done
