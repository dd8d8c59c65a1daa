set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 500 > gpurun_out/mb_clocks.csv &
SMI=$!
./tools/microbench/mma_peak 2>&1 | tee gpurun_out/mma_peak.txt
python tools/microbench/cublas_dgemm.py 2>&1 | tee gpurun_out/cublas_dgemm.txt
kill $SMI
nproc; lscpu | head -20
python -c "import numpy; numpy.show_config()" 2>&1 | tail -30
