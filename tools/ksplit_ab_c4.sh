#!/bin/bash
# A/B of the INT8 kernel's K split at config 4 (n = 16384, K = 16384), same
# box: no split (the default at this K) against ranges of 8192 and 4096.
set -e
mkdir -p gpurun_out
run() {  # $1 = kmax, $2 = tag
  python -c "
import runpy, sys
sys.path.insert(0, '.')
from paper_2008_11480_b200 import _lib
_lib.call('si_ozaki_tune_ksplit', $1)
sys.argv = ['bench.py', '--config', 'c4', '--steps', '5', '--warmup', '3', '--no-e2e', '--no-cpu', '--no-dmma-side']
runpy.run_path('bench.py', run_name='__main__')
" > gpurun_out/ksplit_c4_$2.json 2> gpurun_out/ksplit_c4_$2.err
  python -c "
import json
d = json.loads(open('gpurun_out/ksplit_c4_$2.json').read().strip().splitlines()[-1])
print('$2', d['value'], d['ms_per_step'], d['roofline']['achieved'], d['roofline']['frac'], d['clocks'])
"
}
run 16384 k16384_a
run 8192 k8192_a
run 4096 k4096_a
run 16384 k16384_b
run 8192 k8192_b
run 4096 k4096_b
