# full ncu of the C4 env step (bool mask) with SASS source, to find its instruction hot spots
mkdir -p gpurun_out
timeout 300 python tools/ncu_step.py --game connect_four --batch 4194304 > gpurun_out/step_c4.json 2>&1; echo "plain rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"^lx_env_step\$" -s 3 -c 1 \
   -o gpurun_out/envstep_c4 python tools/ncu_step.py --game connect_four --batch 4194304 > gpurun_out/ncu_envstep.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/envstep_c4.ncu-rep --page raw --csv > gpurun_out/envstep_c4_raw.csv 2>/dev/null
ncu -i gpurun_out/envstep_c4.ncu-rep --page source --csv --print-source sass > gpurun_out/envstep_c4_sass.csv 2>/dev/null
ncu -i gpurun_out/envstep_c4.ncu-rep --page details --csv > gpurun_out/envstep_c4_details.csv 2>/dev/null
rm -f gpurun_out/*.ncu-rep
ls -la gpurun_out | tail -5
