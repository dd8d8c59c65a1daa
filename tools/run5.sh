cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python tools/profile_gemm.py 16384 2 > gpurun_out/r5_plain.log 2>&1 && \
ncu --set full --clock-control none -k regex:gemm_f64_tma -s 1 -c 1 -o gpurun_out/gemm_full_16384_r01 python tools/profile_gemm.py 16384 2 > gpurun_out/r5_ncu.log 2>&1
tail -1 gpurun_out/r5_ncu.log
for c in c1 c2 c3; do timeout 600 python bench.py --config $c --no-cpu > gpurun_out/r5_bench_$c.json 2>gpurun_out/r5_bench_$c.err; tail -1 gpurun_out/r5_bench_$c.json; tail -2 gpurun_out/r5_bench_$c.err; done
timeout 1200 python bench.py --config c5 --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/r5_bench_c5.json 2>gpurun_out/r5_bench_c5.err; tail -1 gpurun_out/r5_bench_c5.json; tail -3 gpurun_out/r5_bench_c5.err
nvidia-smi --query-gpu=memory.used,memory.total --format=csv
