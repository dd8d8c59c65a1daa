cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
for c in c1 c2; do timeout 600 python bench.py --config $c --no-cpu > gpurun_out/r6_bench_$c.json 2>gpurun_out/r6_bench_$c.err; tail -1 gpurun_out/r6_bench_$c.json | cut -c1-600; tail -2 gpurun_out/r6_bench_$c.err; done
timeout 1500 python bench.py --config c5 --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/r6_bench_c5.json 2>gpurun_out/r6_bench_c5.err; tail -1 gpurun_out/r6_bench_c5.json | cut -c1-900; tail -3 gpurun_out/r6_bench_c5.err
