# ncu of the C4 per-ply kernels on the current build (env step bool / bits, random step) with SASS
mkdir -p gpurun_out
timeout 300 python tools/ncu_step.py --game connect_four --batch 4194304 > gpurun_out/step_c4.json 2>&1; echo "plain rc=$?"
for spec in "lx_env_step:3:envbool" "lx_env_step:8:envbits" "lx_random_step:2:rstep"; do
  k=${spec%%:*}; rest=${spec#*:}; skip=${rest%%:*}; tag=${rest#*:}
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:"^$k\$" -s $skip -c 1 \
     -o gpurun_out/p_$tag python tools/ncu_step.py --game connect_four --batch 4194304 > gpurun_out/ncu_$tag.log 2>&1; echo "$tag rc=$?"
  ncu -i gpurun_out/p_$tag.ncu-rep --page details --csv > gpurun_out/${tag}_details.csv 2>/dev/null
  ncu -i gpurun_out/p_$tag.ncu-rep --page source --csv --print-source sass > gpurun_out/${tag}_sass.csv 2>/dev/null
done
rm -f gpurun_out/*.ncu-rep
