cd $GRAFT_REPO_ROOT
python tools/profile_gemm.py 8192 3 > gpurun_out/r2_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gemm_f64_tma -s 1 -c 1 -o gpurun_out/gemm_full_r01 python tools/profile_gemm.py 8192 3 > gpurun_out/r2_ncu_full.log 2>&1
tail -3 gpurun_out/r2_ncu_full.log
python bench.py > gpurun_out/r2_bench_plain.json 2>gpurun_out/r2_bench_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4_r01.csv python bench.py > gpurun_out/r2_ncu_launch.log 2>&1
tail -2 gpurun_out/r2_ncu_launch.log; cat gpurun_out/r2_bench_plain.json
