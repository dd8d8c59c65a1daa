cd $GRAFT_REPO_ROOT
python tools/gemm_bench.py 1024 2048 4096 8192 16384 2>&1 | tee gpurun_out/r4_gemm_bench.txt
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python tools/profile_gemm.py 8192 3 > gpurun_out/r4_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gemm_f64_tma -s 1 -c 1 -o gpurun_out/gemm_full_r01c python tools/profile_gemm.py 8192 3 > gpurun_out/r4_ncu_full.log 2>&1
tail -1 gpurun_out/r4_ncu_full.log
python bench.py --no-cpu > gpurun_out/r4_bench.json 2>&1; tail -1 gpurun_out/r4_bench.json
