for rep in 1 2; do
for g in connect_four tic_tac_toe pente; do
  for t in . _ab/r1h; do
    (cd $t && timeout 300 python tools/ab_rollout.py --game $g --batch 4194304 --reps 10 | sed "s|^|$t |") >> gpurun_out/ab.txt 2>&1
  done
done; done
