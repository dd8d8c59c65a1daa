"""Row-panel exchange over peer memory (peer.py, si_gemm_panels) on one GPU.

* kernel level: a product whose right operand's row panels are still being
  copied (copy engine, flags by stream memory operations) waits for each panel
  inside the DMMA kernel and equals the ungated product bitwise;
* engine level: P virtual ranks in one process (LocalFabric, mode "stream":
  nothing spins on the SMs) run the block-row sharded steps and match the
  single-GPU native steps bitwise, counters included.
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _gemm(a, b, c=None, gate=None, alpha=1.0, beta=0.0, diag=0.0, stream=None):
    from paper_2008_11480_b200 import _lib

    m, k = a.shape
    n = b.shape[1]
    out = torch.empty((m, n), dtype=torch.float64, device="cuda")
    buf = _lib.counter_buf()
    sp = (stream or torch.cuda.current_stream()).cuda_stream
    h = _lib.handle(0)
    cp = c.data_ptr() if c is not None else None
    if gate is None:
        _lib.call("si_gemm_ex", h, m, n, k, alpha, a.data_ptr(), k, b.data_ptr(), n, beta, cp, n,
                  diag, 0, out.data_ptr(), n, 0, buf, sp)
    else:
        flags, epoch, bounds = gate
        _lib.call("si_gemm_panels", h, m, n, k, alpha, a.data_ptr(), k, b.data_ptr(), n, beta, cp,
                  n, diag, 0, out.data_ptr(), n, flags.data_ptr(), epoch,
                  _lib.i64_array(bounds), len(bounds) - 1, 0, buf, sp)
    return out, (buf[0], buf[1])


@pytest.mark.parametrize("n,npanels", [(1024, 4), (640, 3), (96, 2)])
def test_gemm_panels_waits_for_late_panels(n, npanels):
    """The consumer is launched before any panel has arrived; the copy stream
    first runs a long dummy copy, then lands panel by panel and raises each
    flag.  n=96 takes the stream-wait path (no TMA kernel)."""
    from paper_2008_11480_b200 import _lib

    torch.manual_seed(0)
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b_true = torch.randn(n, n, dtype=torch.float64, device="cuda")
    c = torch.randn(n, n, dtype=torch.float64, device="cuda")
    ref, _ = _gemm(a, b_true, c=c, alpha=-1.0, beta=1.0, diag=1.0)
    b_buf = torch.zeros_like(b_true)
    flags = torch.zeros(16, dtype=torch.int32, device="cuda")
    bounds = [round(i * n / npanels) for i in range(npanels + 1)]
    big = torch.empty(64 << 20, dtype=torch.float64, device="cuda")  # 512 MB of delay
    big_dst = torch.empty_like(big)
    torch.cuda.synchronize()
    s_main, s_copy = torch.cuda.Stream(), torch.cuda.Stream()
    h = _lib.handle(0)
    out, ctr = _gemm(a, b_buf, c=c, gate=(flags, 7, bounds), alpha=-1.0, beta=1.0, diag=1.0,
                     stream=s_main)
    with torch.cuda.stream(s_copy):
        big_dst.copy_(big)
        for p in reversed(range(npanels)):  # out of order on purpose
            r0, r1 = bounds[p], bounds[p + 1]
            b_buf[r0:r1].copy_(b_true[r0:r1])
            _lib.call("si_stream_write_u32", h, flags.data_ptr() + 4 * p, 7, s_copy.cuda_stream)
    torch.cuda.synchronize()
    assert ctr == (1, 0)
    assert torch.equal(out, ref)


def test_gemm_panels_epoch_compare_wraps():
    """ready iff (int32)(flag - epoch) >= 0: flag 0 satisfies epoch 2^32-1 + 1."""
    torch.manual_seed(1)
    n = 256
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    flags = torch.zeros(16, dtype=torch.int32, device="cuda")
    flags[:2] = torch.tensor([5, 3], dtype=torch.int32)
    out, _ = _gemm(a, b, gate=(flags, 3, [0, 100, n]))  # 5 >= 3, 3 >= 3
    ref, _ = _gemm(a, b)
    assert torch.equal(out, ref)


def test_gemm_panels_rejects_bad_bounds():
    from paper_2008_11480_b200 import _lib

    n = 128
    a = torch.zeros(n, n, dtype=torch.float64, device="cuda")
    flags = torch.zeros(16, dtype=torch.int32, device="cuda")
    for bounds in ([0, 64], [0, 80, 60, n], [1, n], list(range(17)) + [n]):  # last: 17 panels
        with pytest.raises(ValueError):
            _gemm(a, a, gate=(flags, 1, bounds))
    flags.fill_(1)
    out, _ = _gemm(a, a, gate=(flags, 1, list(range(0, n + 1, 8))))  # 16 panels: the maximum
    assert torch.equal(out, torch.zeros_like(a))
    del _lib


def _virtual_ranks(n, world, mode="stream"):
    from paper_2008_11480_b200.peer import LocalFabric, PeerComm
    from paper_2008_11480_b200.sharded import ShardedEngine

    fab = LocalFabric(torch.device("cuda", 0), world)
    engs = [ShardedEngine(PeerComm(n, fab.view(r), mode=mode)) for r in range(world)]
    streams = [torch.cuda.Stream() for _ in range(world)]
    return engs, streams


@pytest.mark.parametrize("world,n", [(2, 384), (3, 384), (3, 386), (4, 200)])
def test_virtual_ranks_composite_step_bitwise(world, n, monkeypatch):
    """composite_step (newton_schulz.py:177-228) on P block-row virtual ranks
    exchanging panels over the peer path equals the native single-GPU step
    (uneven splits: 386 = 129 + 129 + 128, panel bounds off the 16-row k-slabs;
    n = 200: row blocks of 50 below the DMMA kernel's 128-row tiles)."""
    import paper_2008_11480_b200 as P

    rng = np.random.default_rng(5)
    g = rng.standard_normal((2 * n, n))
    a_np = g.T @ g / (2 * n) + 0.5 * np.eye(n)
    a = torch.as_tensor(a_np, device="cuda")
    sp = P.split_scalar(a, P.inf_norm(a) / 2.0, check_pd=False, verify=False)
    st = P.initial_series(sp, 0, 1, order=2)
    spec = P.CompositeSpec((2, 3, 4, 5))
    ref = P.composite_step(st, a, sp, spec, 2)
    ref2 = P.composite_step(ref, a, sp, spec, 2)

    monkeypatch.setenv("SI_PEER_CHECK", "1")  # every rank pairs every gather with the same slot
    engs, streams = _virtual_ranks(n, world)
    outs = []
    for r, (eng, s) in enumerate(zip(engs, streams)):
        c = eng.comm
        with torch.cuda.stream(s):
            s.wait_stream(torch.cuda.default_stream())
            A, Pm, B = eng.replicated(a), eng.replicated(sp.precond), eng.replicated(sp.residual)
            gr = eng.local(st.estimate[c.r0:c.r1].clone())
            fr = eng.local(st.residual[c.r0:c.r1].clone())
            for _ in range(2):
                gr, fr = eng.composite_step(gr, fr, A, Pm, B, (2, 3, 4, 5), 2)
            outs.append((gr, fr))
    torch.cuda.synchronize()
    g_cat = torch.cat([eng.rows_of(o[0]) for eng, o in zip(engs, outs)])
    f_cat = torch.cat([eng.rows_of(o[1]) for eng, o in zip(engs, outs)])
    assert torch.equal(g_cat, ref2.estimate)
    assert torch.equal(f_cat, ref2.residual)
    for eng in engs:
        assert eng.ctr.mmm == 2 * 22
        assert eng.comm.bytes_gathered > 0
        # products are written straight into their exchange slots; copied in are
        # only the first step's input G and, per step, the one part whose plan
        # ends in a Lin (not a product)
        assert eng.comm.local_copies <= 1 + 2


def test_virtual_ranks_recursive_step_bitwise():
    """richardson_recursive_step (richardson.py:111-189) incl. the n x 1 theta
    exchanges on 2 virtual ranks equals the block-row engine over NCCL-free
    single rank (itself bitwise the native step, test_gpu_parity)."""
    from paper_2008_11480_b200.sharded import RowComm, ShardedEngine

    n, order, world = 256, 4, 2
    rng = np.random.default_rng(9)
    g = rng.standard_normal((2 * n, n))
    a_np = g.T @ g / (2 * n) + 0.5 * np.eye(n)
    alpha = float(np.abs(a_np).sum(axis=1).max())
    a = torch.as_tensor(a_np, device="cuda")
    b = torch.as_tensor(rng.standard_normal((n, 1)), device="cuda")
    eye = torch.eye(n, dtype=torch.float64, device="cuda")
    g0, f0 = eye / alpha, eye - a / alpha
    l0, r0m = g0.clone(), f0.clone()
    theta0 = torch.zeros_like(b)

    def run(eng, rows):
        A, bb = eng.replicated(a), eng.replicated(b)
        st = [eng.local(m[rows].clone()) for m in (g0, f0, l0, r0m)] + [None, None]
        th = eng.replicated(theta0)
        for _ in range(2):
            gg, ff, ll, rr, om, ns, th = eng.richardson_recursive_step(
                st[0], st[1], st[2], st[3], st[4], st[5], A, th, bb, order)
            st = [gg, ff, ll, rr, om, ns]
        return eng.rows_of(st[0]), th.t

    single = ShardedEngine(RowComm(n))
    g_ref, th_ref = run(single, slice(0, n))
    engs, streams = _virtual_ranks(n, world)
    outs = []
    for eng, s in zip(engs, streams):
        with torch.cuda.stream(s):
            s.wait_stream(torch.cuda.default_stream())
            outs.append(run(eng, slice(eng.comm.r0, eng.comm.r1)))
    torch.cuda.synchronize()
    assert torch.equal(torch.cat([o[0] for o in outs]), g_ref)
    for o in outs:
        assert torch.equal(o[1], th_ref)
    assert all(e.ctr.mmm == single.ctr.mmm and e.ctr.mvm == single.ctr.mvm for e in engs)


def test_slot_reuse_across_steps_is_bounded():
    """Exchange slots are leased while a gathered value lives and reused after:
    ten steps must not grow the slot pool beyond the first step's."""
    import paper_2008_11480_b200 as P

    n, world = 256, 2
    rng = np.random.default_rng(3)
    g = rng.standard_normal((2 * n, n))
    a = torch.as_tensor(g.T @ g / (2 * n) + 0.5 * np.eye(n), device="cuda")
    sp = P.split_scalar(a, P.inf_norm(a) / 2.0, check_pd=False, verify=False)
    st = P.initial_series(sp, 0, 1, order=2)
    engs, streams = _virtual_ranks(n, world)
    states = []
    for eng in engs:
        c = eng.comm
        states.append([eng.local(st.estimate[c.r0:c.r1].clone()),
                       eng.local(st.residual[c.r0:c.r1].clone())])
    sizes = []
    for step in range(10):
        for r, (eng, s) in enumerate(zip(engs, streams)):
            with torch.cuda.stream(s):
                s.wait_stream(torch.cuda.default_stream())
                A, Pm, B = eng.replicated(a), eng.replicated(sp.precond), eng.replicated(sp.residual)
                states[r] = list(eng.composite_step(states[r][0], states[r][1], A, Pm, B,
                                                    (2, 3), 2))
        sizes.append(len(engs[0].comm._slots))
    torch.cuda.synchronize()
    assert sizes[-1] == sizes[0]
    assert len({len(e.comm._slots) for e in engs}) == 1


def test_ipc_processes_composite_step(tmp_path):
    """Two processes on the one GPU exchange row panels through CUDA IPC
    mappings (IpcFabric: si_sym_alloc / si_sym_open, flags written into the
    peer's mapping, copy-engine pulls from it); mode "stream", so no kernel
    waits on the other process.  Three composite steps equal the native
    single-GPU steps bitwise."""
    import os
    import socket
    import subprocess
    import sys

    import paper_2008_11480_b200 as P

    from conftest import release_gpu_memory

    release_gpu_memory()
    n, world = 384, 2
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = str(s.getsockname()[1])
    worker = os.path.join(os.path.dirname(os.path.abspath(__file__)), "peer_ipc_worker.py")
    procs = [subprocess.Popen([sys.executable, worker, str(r), str(world), port, str(tmp_path),
                               str(n)]) for r in range(world)]
    try:
        codes = [p.wait(timeout=240) for p in procs]
    finally:
        for p in procs:
            if p.poll() is None:
                p.kill()
    assert codes == [0] * world

    rng = np.random.default_rng(5)
    g = rng.standard_normal((2 * n, n))
    a = torch.as_tensor(g.T @ g / (2 * n) + 0.5 * np.eye(n), device="cuda")
    sp = P.split_scalar(a, P.inf_norm(a) / 2.0, check_pd=False, verify=False)
    st = P.initial_series(sp, 0, 1, order=2)
    spec = P.CompositeSpec((2, 3, 4, 5))
    for _ in range(3):
        st = P.composite_step(st, a, sp, spec, 2)
    from paper_2008_11480_b200.sharded import row_splits

    gs, fs = [], []
    for r, (r0, r1) in enumerate(row_splits(n, world)):
        blk = np.load(tmp_path / f"rank{r}.npy")
        gs.append(blk[:r1 - r0])
        fs.append(blk[r1 - r0:])
        mmm, slots = np.load(tmp_path / f"ctr{r}.npy")
        assert mmm == 3 * 22
    assert np.array_equal(np.concatenate(gs), st.estimate.cpu().numpy())
    assert np.array_equal(np.concatenate(fs), st.residual.cpu().numpy())
