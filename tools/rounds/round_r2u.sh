# small-batch latency: fixed vs per-ply cost of lx_rollout at B=1024; bench per-config with
# the add-free graphs
mkdir -p gpurun_out
for g in tic_tac_toe connect_four; do
  timeout 300 python tools/latency_probe.py --game $g --batch 1024 --caps 0,1,2,3,4,5,6,7,8,9,12,16,24,200 > gpurun_out/lat_$g.jsonl 2>&1; echo "$g rc=$?"
done
timeout 300 python tools/latency_probe.py --game tic_tac_toe --batch 32 --caps 0,1,9,200 > gpurun_out/lat_ttt32.jsonl 2>&1
cat gpurun_out/lat_*.jsonl
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench rc=$?"; tail -c 300 gpurun_out/bench_c4.err
