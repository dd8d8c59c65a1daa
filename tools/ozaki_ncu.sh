#!/bin/bash
# ncu captures of the Ozaki-II kernels at n=16384 (one emulated product):
# launch list (shares) and --set full of the INT8 pair kernel, the CRT and the
# residue kernels.  Run under gpurun; the plain run must exit 0 first.
set -e
mkdir -p gpurun_out
python tools/ozaki_one.py 16384 16
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/ozaki_launches.csv python tools/ozaki_one.py 16384 16 > /dev/null
ncu --set full --clock-control none --import-source on -k regex:'i8_gemm|crt|residues|absmax' \
    -c 6 -o gpurun_out/oz_full python tools/ozaki_one.py 16384 16 > gpurun_out/ncu_oz.log 2>&1
