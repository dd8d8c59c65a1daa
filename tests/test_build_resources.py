"""Resource usage of the hot kernels in the built library (cuobjdump, no GPU
needed): a stack frame in one of them means an accumulator / fragment array
went to local memory -- the regression that once cost the INT8 kernel 7%
(a run-time flag made its epilogue index v[32] dynamically)."""

import os
import re
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2008_11480_b200", "libseriesinv_b200.so")

# mangled-name fragment -> (max registers, max stack bytes)
LIMITS = {
    "gemm_f64_tma_kernel": (232, 0),           # DMMA GEMM: 128 FP64 accumulators per consumer thread
    "i8_gemm_mod_kernelILb0": (96, 32),        # default INT8 kernel (32 B: the ragged byte-store path)
    "crt_kernelILi16": (80, 0),
    "residues_rows_kernel": (64, 0),
    "resident_kernelILi32": (128, 0),          # config-2 resident kernels (<= 4 CTAs x 128 threads / SM)
}


def _usage():
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        pytest.skip("cuobjdump not available")
    if not os.path.exists(LIB):
        pytest.skip("library not built")
    out = subprocess.run([exe, "--dump-resource-usage", LIB], capture_output=True, text=True,
                         check=True).stdout
    res, name = {}, None
    for line in out.splitlines():
        m = re.search(r"Function (\S+):", line)
        if m:
            name = m.group(1)
            continue
        m = re.search(r"REG:(\d+) STACK:(\d+)", line)
        if m and name:
            res[name] = (int(m.group(1)), int(m.group(2)))
            name = None
    return res


def test_hot_kernels_keep_their_arrays_in_registers():
    res = _usage()
    assert res, "no kernels found in the library"
    for frag, (max_reg, max_stack) in LIMITS.items():
        hits = {k: v for k, v in res.items() if frag in k}
        assert hits, f"kernel {frag} not found"
        for k, (reg, stack) in hits.items():
            assert reg <= max_reg and stack <= max_stack, (k, reg, stack)
