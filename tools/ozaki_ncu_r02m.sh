#!/bin/bash
# Final-state captures of the default INT8 kernel (single CTA, 4-stage ring,
# GROUP_M 16): --set full at n=16384 (one emulated product), and DRAM bytes /
# tensor pipe of the kernel at n = 4096 and 32768 (the C3 / C5 product shapes).
# Run under gpurun; each plain run exits 0 first.
set -e
mkdir -p gpurun_out
M="dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_tensor.sum,lts__t_sector_hit_rate.pct,sm__cycles_active.avg"
for n in 4096 16384 32768; do
  python tools/ozaki_one.py $n 16
  ncu --metrics $M --clock-control none -k regex:i8_gemm_mod -s 1 -c 3 --csv \
      --log-file gpurun_out/ncu_i8_dram_$n.csv python tools/ozaki_one.py $n 16 > /dev/null
done
ncu --set full --clock-control none --import-source on -k regex:i8_gemm_mod -s 1 -c 1 \
    -o gpurun_out/i8_full_r02m python tools/ozaki_one.py 16384 16 > gpurun_out/ncu_i8_full.log 2>&1
ncu -i gpurun_out/i8_full_r02m.ncu-rep --page raw --csv > gpurun_out/i8_full_r02m_raw.csv
