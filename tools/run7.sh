cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -4
timeout 600 python bench.py --config c1 --no-cpu > gpurun_out/r7_bench_c1.json 2>gpurun_out/r7_bench_c1.err; tail -1 gpurun_out/r7_bench_c1.json | cut -c1-700; tail -2 gpurun_out/r7_bench_c1.err
cat > gpurun_out/r7_c2prof.py <<'PY'
import sys, torch
sys.path.insert(0, ".")
import paper_2008_11480_b200 as P
from paper_2008_11480_b200 import configs
a_np, b_np = configs.c2_batched(batch=2048)
a, b = P.as_device(a_np), P.as_device(b_np)
pre, res = P.batched_scalar_split(a)
for _ in range(2):
    P.batched_composite_richardson(a, b, pre, res, pre, res, torch.zeros_like(b), (2, 3), 2, 10)
torch.cuda.synchronize(); print("ok")
PY
python gpurun_out/r7_c2prof.py > gpurun_out/r7_c2_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:resident -s 1 -c 1 -o gpurun_out/resident_c2_r01 python gpurun_out/r7_c2prof.py > gpurun_out/r7_ncu.log 2>&1
tail -1 gpurun_out/r7_ncu.log
