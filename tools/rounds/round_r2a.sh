# r2a: first GPU check of round 2 -- env-step kernel (fused random step, bit
# masks, auto-reset latch, illegal actions), bench per_config block.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_env.py tests/test_gpu_movement.py -q -x > gpurun_out/pytest_env.log 2>&1; tail -3 gpurun_out/pytest_env.log
timeout 900 python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench rc=$?"; tail -c 400 gpurun_out/bench_c4.err
timeout 600 python bench.py --impl reference --steps 20 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout 900 python tools/sweep.py --min-log2 10 --max-log2 22 > gpurun_out/sweep.jsonl 2> gpurun_out/sweep.err; echo "sweep rc=$?"
nproc > gpurun_out/nproc.txt; lscpu > gpurun_out/lscpu.txt
