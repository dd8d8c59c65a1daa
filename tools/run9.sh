cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -k "resident or batched" 2>&1 | tail -15
for c in c1 c2; do timeout 600 python bench.py --config $c --no-cpu > gpurun_out/r9_bench_$c.json 2>gpurun_out/r9_bench_$c.err; tail -1 gpurun_out/r9_bench_$c.json | cut -c1-330; tail -2 gpurun_out/r9_bench_$c.err; done
