#!/bin/bash
# A/B of the INT8 kernel's K split at config 5 (n = 32768), same box: ranges
# of 16384 against no split (the default).
set -e
mkdir -p gpurun_out
run() {  # $1 = kmax, $2 = tag
  python -c "
import runpy, sys
sys.path.insert(0, '.')
from paper_2008_11480_b200 import _lib
_lib.call('si_ozaki_tune_ksplit', $1)
sys.argv = ['bench.py', '--config', 'c5', '--steps', '3', '--warmup', '3', '--no-e2e', '--no-cpu', '--no-dmma-side']
runpy.run_path('bench.py', run_name='__main__')
" > gpurun_out/ksplit_$2.json 2> gpurun_out/ksplit_$2.err
  python -c "
import json
d = json.loads(open('gpurun_out/ksplit_$2.json').read().strip().splitlines()[-1])
print('$2', d['value'], d['ms_per_step'], d['roofline']['achieved'], d['roofline']['frac'], d['clocks'])
"
}
run 0 nosplit
run 16384 split
run 0 nosplit2
run 16384 split2
