cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/r1_pytest_gpu.txt
tail -30 gpurun_out/r1_pytest_gpu.txt
timeout 300 python __graft_entry__.py > gpurun_out/r1_smoke.txt 2>&1; tail -5 gpurun_out/r1_smoke.txt
timeout 600 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu > gpurun_out/r1_bench_c3.json 2> gpurun_out/r1_bench_c3.err; cat gpurun_out/r1_bench_c3.json; tail -5 gpurun_out/r1_bench_c3.err
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/r1_bench_c4.json 2> gpurun_out/r1_bench_c4.err; cat gpurun_out/r1_bench_c4.json; tail -5 gpurun_out/r1_bench_c4.err
