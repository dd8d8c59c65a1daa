cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3
for c in c1 c2; do timeout 600 python bench.py --config $c --no-cpu > gpurun_out/r8_bench_$c.json 2>gpurun_out/r8_bench_$c.err; tail -1 gpurun_out/r8_bench_$c.json | cut -c1-420; tail -2 gpurun_out/r8_bench_$c.err; done
