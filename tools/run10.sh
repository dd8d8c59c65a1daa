cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
python tools/c2prof.py > gpurun_out/r10_c2_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:resident -s 1 -c 1 -o gpurun_out/resident_c2_r01b python tools/c2prof.py > gpurun_out/r10_ncu.log 2>&1
tail -1 gpurun_out/r10_ncu.log
