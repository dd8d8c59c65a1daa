cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -k "resident or batched or hoisted" 2>&1 | tail -2
for c in c1 c2; do timeout 600 python bench.py --config $c --no-cpu > gpurun_out/r12_bench_$c.json 2>gpurun_out/r12_bench_$c.err; python -c "import json;d=json.load(open('gpurun_out/r12_bench_$c.json'));print('$c', d['value'], d['tflops'], d['tflops_frac_of_dmma_peak'])"; tail -2 gpurun_out/r12_bench_$c.err; done
timeout 600 python bench.py --hoist --no-cpu > gpurun_out/r12_bench_c4h.json 2>gpurun_out/r12_bench_c4h.err; python -c "import json;d=json.load(open('gpurun_out/r12_bench_c4h.json'));print('c4 hoisted', d['value'], d['tflops'], d['tflops_frac_of_dmma_peak'])"; tail -2 gpurun_out/r12_bench_c4h.err
python tools/c2prof.py > gpurun_out/r12_c2_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:resident -s 1 -c 1 -o gpurun_out/resident_c2_r01c python tools/c2prof.py > gpurun_out/r12_ncu.log 2>&1
tail -1 gpurun_out/r12_ncu.log
