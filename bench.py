"""Benchmark of the seriesinv B200 hot path (BASELINE.json metric).

Default workload = BASELINE config 4: dense SPD n=16384 (Householder-product
eigenbasis, lambda log-uniform in [1, 1e6]), 64 right-hand sides; one step =
one plain Richardson update with P_k + one composite Newton-Schulz
step with rates (2,3,4,5), order_n=2 (newton_schulz.py:177-228) -- the
reference GEMM DAG, 22 n^3 products + 2 n^2 r products, recomputed every step.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c1|c2|c3|c4|c5] [--n N]

Prints ONE JSON line on rank 0.  Timing: CUDA events on the launching stream,
barrier + synchronize on both sides, max over ranks; inputs (2.1 GB per matrix)
are far larger than the 126 MB L2, so no flush is needed.
"""

from __future__ import annotations

import argparse
import json
import os

# the sharded path's exchange streams wait on flags: give every stream its own
# hardware work queue (paper_2008_11480_b200/peer.py); before CUDA initialises
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
SHARE_GPU = os.environ.get("SI_BENCH_SHARE_GPU") == "1"
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "iters/s and FP64 TFLOP/s (% of peak) of composite Newton-Schulz at n=16384"


# --------------------------------------------------------------------------- helpers


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap,power.draw")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm, smax, reasons, power = [], [], set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
                power.append(float(parts[6]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {
            "sm_mhz": statistics.median(sm) if sm else None,
            "sm_max_mhz": max(smax) if smax else None,
            "reasons": sorted(reasons),
            "samples": len(sm),
            "power_w_median": statistics.median(power) if power else None,
        }


def dist_setup(args):
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and SHARE_GPU:
        # test mode (SI_BENCH_SHARE_GPU=1): every rank on cuda:0, gloo for the
        # host-side collectives; exercises the N > 1 code paths on a 1-GPU box
        # (timings are meaningless: the ranks share one GPU)
        import torch.distributed as dist

        torch.cuda.set_device(0)
        dist.init_process_group("gloo")
        return world, rank, 0
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    elif torch.cuda.is_available():
        torch.cuda.set_device(0)
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cpu" if SHARE_GPU else "cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def ncu_traffic(w) -> float | None:
    """DRAM bytes per launch of the dominant kernel at this workload's n, from the
    committed ncu --set full capture (profiles/ncu_traffic.json), else None."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as fh:
            data = json.load(fh)
        rec = data.get("gemm_f64_tma_kernel", {}).get(str(w.n))
        return float(rec["dram_bytes_per_launch"]) if rec else None
    except (OSError, ValueError, KeyError):
        return None


def l2_note(w) -> str:
    """How the timed region relates to the 126 MB L2 (timing rule: inputs larger
    than L2, or a flush)."""
    if w.cfg == "c1":
        return ("no flush: one launch runs 30 iterations out of shared memory/DSMEM; "
                "its inputs (a few 64x64 matrices) are read once per launch (latency-bound config)")
    if w.cfg == "c2":
        return (f"inputs larger than L2 ({8 * w.batch * w.n * w.n / 1e6:.0f} MB per "
                f"{w.batch}x{w.n}^2 stack, read once per launch), no flush")
    return f"inputs larger than L2 ({8 * w.n * w.n / 1e9:.2f} GB per n x n matrix), no flush"


def resident_roofline(w, tflops_per_gpu: float, step_s: float, peak: float) -> dict:
    """Configs 1/2: one resident_kernel launch per step (the whole timed region), so
    the kernel's achieved rate is the step's; HBM bytes are algorithmic: per system
    A, S^-1, F, P in + P, F out (n^2 doubles each), b, theta, and S^-1, B streamed
    in every iteration (config 2)."""
    n = w.n
    systems = w.batch if w.cfg == "c2" else 1
    per_sys = 8 * (6 * n * n + 3 * n)
    if w.cfg == "c2":
        per_sys += 8 * 2 * n * n * w.iters_per_step
    gbs = systems * per_sys / step_s / 1e9
    return {"bound": "tensor" if w.cfg == "c2" else "latency", "achieved": tflops_per_gpu,
            "peak": peak, "unit": "TFLOP/s", "frac": tflops_per_gpu / peak, "traffic": None,
            "kernel": "resident_kernel<32>" if w.cfg == "c2" else "resident_kernel<64>",
            "hbm_gbs_algorithmic": gbs,
            "peak_source": "measured live: DMMA m8n8k4 register-only probe (si_dmma_peak)"}


def dmma_side_run(w, args, h, flops: float, peak: float) -> dict:
    """The same workload with every product on FP64 DMMA (the library default),
    timed right after the emulated run in the same process: a few steps, CUDA
    events, clocks sampled -- the FP64-tensor-core reference point of the line."""
    import ctypes

    import torch

    from paper_2008_11480_b200 import _lib

    k = 1 if w.cfg == "c5" else max(1, min(args.steps, 3))  # c5: ~35 s per DMMA step
    with w.P.gemm_backend("dmma"):
        w.step()  # warm (kernels, workspace)
        torch.cuda.synchronize()
        sampler = ClockSampler(int(os.environ.get("LOCAL_RANK", "0")))
        sampler.start()
        _lib.call("si_profile_begin", h)
        stream = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(k):
            w.step()
        e1.record(stream)
        torch.cuda.synchronize()
        g_ms, g_fl = ctypes.c_double(), ctypes.c_double()
        g_n, launches = ctypes.c_int64(), ctypes.c_int64()
        _lib.call("si_profile_end", h, ctypes.byref(g_ms), ctypes.byref(g_fl), ctypes.byref(g_n),
                  ctypes.byref(launches))
        clocks = sampler.stop()
    step_s = e0.elapsed_time(e1) / 1e3 / k
    ach = g_fl.value / (g_ms.value / 1e3) / 1e12 if g_ms.value > 0 else None
    return {"what": "same workload, every product on FP64 DMMA (gemm_f64_tma_kernel), timed after "
                    "the emulated run in this process",
            "value": w.iters_per_step / step_s, "unit": "iters/s", "steps": k,
            "ms_per_step": step_s * 1e3, "tflops": flops / step_s / 1e12,
            "roofline": {"bound": "tensor", "achieved": ach, "peak": peak, "unit": "TFLOP/s",
                         "frac": ach / peak if ach else None, "kernel": "gemm_f64_tma_kernel",
                         "launches": g_n.value,
                         "peak_source": "measured live: DMMA register-only probe (si_dmma_peak)"},
            "clocks": clocks}


def int8_peak_tops() -> tuple[float, str]:
    """Measured INT8 tensor-core yardstick: cuBLASLt int8 GEMM 8192^3
    (torch._int_mm, int8 x int8 -> int32), best of 10 launches (burst, like
    MEASURED_PEAKS.json's bf16 figure); MEASURED_PEAKS.json has no INT8 entry."""
    import torch

    n = 8192
    g = torch.Generator(device="cuda").manual_seed(0)
    a = torch.randint(-128, 128, (n, n), dtype=torch.int8, device="cuda", generator=g)
    b = torch.randint(-128, 128, (n, n), dtype=torch.int8, device="cuda", generator=g).t()
    torch._int_mm(a, b)
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch._int_mm(a, b)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    del a, b
    return 2.0 * n**3 / (best * 1e-3) / 1e12, (
        "measured live before the timed region: cuBLASLt int8 GEMM 8192^3 (torch._int_mm), "
        "best of 10 (burst); MEASURED_PEAKS.json has no INT8 entry (nominal dense INT8: 4500 TOPS)")


def ozaki_roofline(w, i8_ms: float, i8_ops: float, i8_launches: int, fp64_achieved, fp64_launches,
                   dmma_peak: float, moduli: int, i8_peak: tuple) -> dict:
    """Roofline of the Ozaki-II products: the dominant kernel is the INT8
    tcgen05 GEMM (i8_gemm_mod_kernel); achieved = its algorithmic int8 ops
    (2 M N Kp per modulus plane) / its CUDA-event time on the launching stream."""
    peak, src = i8_peak
    ach = i8_ops / (i8_ms * 1e-3) / 1e12 if i8_ms > 0 else None
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            rec = json.load(fh).get("i8_gemm_mod_kernel", {}).get(str(w.n))
        traffic = float(rec["dram_bytes_per_launch"]) if rec else None
    except (OSError, ValueError, KeyError):
        pass
    return {"bound": "tensor", "achieved": ach, "peak": peak, "unit": "TOPS (int8)",
            "frac": ach / peak if ach else None, "traffic": traffic,
            "kernel": {"pair": "i8_gemm_mod_pair_kernel", "multicast": "i8_gemm_mod_mc_kernel"}.get(
                getattr(w, "i8_kernel", "auto"), "i8_gemm_mod_kernel"),
            "launches": i8_launches, "moduli": moduli,
            "peak_source": src,
            "fp64_equivalent": {
                "what": "whole emulated products (scaling, residues, INT8 GEMM, CRT + epilogue): "
                        "2 M N K FP64 FLOP / their CUDA-event time",
                "achieved_tflops": fp64_achieved, "launches": fp64_launches,
                "dmma_peak_tflops": dmma_peak,
                "frac_of_dmma_peak": fp64_achieved / dmma_peak if fp64_achieved else None}}


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def use_all_host_threads() -> int:
    """The CPU baseline runs on every host core it may use: torchrun exports
    OMP_NUM_THREADS=1, which would otherwise pin OpenBLAS to one thread."""
    n = host_cores()
    try:
        from threadpoolctl import threadpool_limits

        threadpool_limits(limits=n)
    except ImportError:
        pass
    return n


# --------------------------------------------------------------------------- workloads


def make_comm(n: int, kind: str):
    """Row-panel exchange of the sharded path: "peer" (copy engines over CUDA
    IPC, products gated per panel inside the DMMA kernel), "peer-stream"
    (same transfers, stream waits before each product) or "nccl" (NCCL
    all-gather, the library baseline)."""
    import torch

    from paper_2008_11480_b200.sharded import RowComm

    if kind == "nccl":
        return RowComm(n)
    from paper_2008_11480_b200.peer import IpcFabric, PeerComm

    dev = torch.device("cuda", torch.cuda.current_device())
    if SHARE_GPU:
        # ranks sharing one GPU must not spin in kernels on each other's panels
        kind = "peer-stream"
    # The peer exchange needs CUDA IPC mappings and peer access between every
    # pair of GPUs.  If any rank cannot set it up (no P2P between two devices,
    # IPC disabled in a container), every rank falls back to the NCCL
    # all-gather together and the JSON line says so (``comm_fallback``).
    import torch.distributed as dist

    comm, why = None, ""
    try:
        comm = PeerComm(n, IpcFabric(dev), mode="fused" if kind == "peer" else "stream")
    except Exception as exc:  # noqa: BLE001 -- any set-up failure takes the fallback
        why = f"{type(exc).__name__}: {exc}"[:200]
    ok = torch.tensor([1 if comm is not None else 0], dtype=torch.int32,
                      device="cpu" if SHARE_GPU else dev)
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    if int(ok.item()) == 1:
        return comm
    COMM_FALLBACK["reason"] = why or "peer exchange set-up failed on another rank"
    del comm
    return RowComm(n)


COMM_FALLBACK: dict = {}


_COMM_LABEL = {"peer": "copy-engine panel exchange, panel-gated products",
               "peer-stream": "copy-engine panel exchange, stream-gated products",
               "nccl": "NCCL all-gather",
               "native": "library block-row engine (si_sharded_*), NCCL all-gather"}


def workload_desc(cfg: str, n: int, batch: int = 16384) -> str:
    """The `config.workload` string of a config (both arms print the same one)."""
    if cfg == "c4":
        return (f"c4: dense SPD n={n}, Householder(64) eigenbasis, kappa 1e6, 64 RHS; "
                "composite NS rates (2,3,4,5) order_n=2 + plain Richardson")
    if cfg == "c3":
        return f"c3: Gram n={n}; order-8 factorised NS (h8) + plain Richardson"
    if cfg == "c1":
        return (f"c1: dense SPD n={n}; 30 x (plain Richardson + NS order 3), "
                "resident kernel (one launch per 30-iteration run)")
    if cfg == "c5":
        return f"c5: Gram n={n}, 256 RHS; recursive Richardson/NS order 16"
    if cfg == "c2":
        return (f"c2: {batch} systems 32x32; 50 x (plain Richardson + composite "
                "(2,3) order_n=2), resident kernel (one launch per 50-iteration run)")
    raise ValueError(cfg)


class Workload:
    """One config: device state + one step function + algorithmic FLOPs per step."""

    def __init__(self, cfg: str, n: int | None, world: int = 1, hoist: bool = False,
                 comm: str = "peer", shard: str = "rows"):
        self.cfg = cfg
        self.shard = shard
        self.n = n
        self.world = world
        self.hoist = hoist
        self.comm_kind = comm
        self.sharded = None
        self.native = None
        self.split_batch = False
        self.iters_per_step = 1
        self.executor = None  # composite parts on concurrent streams (--streams)

    # FLOPs of the executed reference DAG per step (2 M N K summed)
    def flops(self) -> float:
        n = self.n
        if self.cfg == "c4":
            # executed DAG: 22 products per step, or 3 with the opt-in hoisted parts
            return (3 if self.hoist else 22) * 2.0 * n**3 + 2 * 2.0 * n * n * self.r
        if self.cfg == "c3":
            return 6 * 2.0 * n**3 + 2 * 2.0 * n * n
        if self.cfg == "c1":
            return self.iters_per_step * (3 * 2.0 * n**3 + 2 * 2.0 * n * n)
        if self.cfg == "c5":
            return self.mmm_per_step * 2.0 * n**3 + 2 * 2.0 * n * n * self.r
        if self.cfg == "c2":
            return self.iters_per_step * self.batch * (10 * 2.0 * 32**3 + 2 * 2.0 * 32 * 32)
        raise ValueError(self.cfg)

    def setup(self):
        import torch

        import paper_2008_11480_b200 as P
        from paper_2008_11480_b200 import configs

        self.P = P
        cfg = self.cfg
        if cfg == "c4":
            self.n = self.n or 16384
            self.r = 64
            if self.n >= 4096:
                a, b = configs.c4_householder_device(n=self.n, rhs=self.r)
            else:
                a, b = (P.as_device(x) for x in configs.c4_householder(n=self.n, rhs=self.r))
            self.workload = workload_desc(cfg, self.n)
        elif cfg == "c3":
            self.n = self.n or 4096
            self.r = 1
            a_np, b_np = configs.c3_gram(n=self.n)
            a, b = P.as_device(a_np), P.as_device(b_np)
            self.workload = workload_desc(cfg, self.n)
        elif cfg == "c1":
            self.n = self.n or 64
            self.r = 1
            a_np, b_np = configs.c1_dense_small(n=self.n)
            a, b = P.as_device(a_np), P.as_device(b_np)
            # one bench step = the whole 30-iteration run in one resident launch
            self.iters_per_step = 30
            self.workload = workload_desc(cfg, self.n)
            alpha = float(torch.max(torch.sum(torch.abs(a), dim=1)))
            eye = torch.eye(self.n, dtype=torch.float64, device=a.device)
            self.c1 = {"a": a, "b": b, "p": eye / alpha, "f": eye - a / alpha,
                       "t": torch.zeros_like(b)}
            self.sharded = None
            return
        elif cfg == "c5":
            self.n = self.n or 32768
            self.r = 256
            a, b = configs.c5_gram_device(n=self.n, m=int(self.n * 40000 / 32768), rhs=self.r)
            self.workload = workload_desc(cfg, self.n)
        elif cfg == "c2":
            self.batch = self.n or 16384
            a_np, b_np = configs.c2_batched(batch=self.batch)
            if self.world > 1:
                # independent systems: each rank takes a contiguous share, no communication
                from paper_2008_11480_b200.sharded import row_splits

                rank = int(os.environ.get("RANK", "0"))
                lo, hi = row_splits(self.batch, self.world)[rank]
                a_np, b_np = a_np[lo:hi], b_np[lo:hi]
                self.split_batch = True
            self.a2, self.b2 = P.as_device(a_np), P.as_device(b_np)
            self.pre2, self.res2 = P.batched_scalar_split(self.a2)
            self.p2, self.f2 = self.pre2.clone(), self.res2.clone()
            self.t2 = torch.zeros_like(self.b2)
            self.iters_per_step = 50
            self.workload = workload_desc(cfg, 32, self.batch)
            self.n = 32
            return
        else:
            raise ValueError(cfg)
        self.a = a
        self.b = b
        # the reference's full setup (splitting.py:124-146, :58-64): fused symmetry
        # check, blocked-Cholesky PD check, the verification product -- untimed
        t_setup = time.perf_counter()
        self.sp = P.split_scalar(a, P.inf_norm(a) / 2.0, check_pd=True, verify=True)
        torch.cuda.synchronize()
        self.setup_s = time.perf_counter() - t_setup
        self.sharded = None
        if self.world > 1 and cfg == "c4" and self.shard == "parts":
            # composite parts on GPU groups + one ordered (t, r) tree reduction
            # (grouped.py); the state is block-row sharded over all ranks
            from paper_2008_11480_b200.grouped import GroupedComposite

            gc = GroupedComposite(self.n, (2, 3, 4, 5), 2)
            eng, comm = gc.eng, gc.comm
            st = P.initial_series(self.sp, 0, 1, order=2)
            self.sharded = {
                "gc": gc, "eng": eng, "comm": comm,
                "A": eng.replicated(self.sp.matrix), "P": eng.replicated(self.sp.precond),
                "B": eng.replicated(self.sp.residual), "b": eng.replicated(b),
                "g": eng.local(st.estimate[comm.r0:comm.r1].clone()),
                "f": eng.local(st.residual[comm.r0:comm.r1].clone()),
                "theta": eng.replicated(torch.zeros_like(b)),
            }
            del st
            torch.cuda.empty_cache()
            self.spec = P.CompositeSpec((2, 3, 4, 5))
            self.workload += (f" [parts on {len(gc.groups)} GPU groups "
                              f"{[len(g) for g in gc.groups]}, segments {gc.segments}]")
            return
        if self.world > 1 and cfg in ("c4", "c3", "c5") and self.comm_kind == "native":
            # the same block-row DAG orchestrated inside the library (si_sharded_*,
            # NCCL all-gathers; on a shared GPU the host exchange)
            from paper_2008_11480_b200 import native_sharded as NS

            comm = NS.NativeComm.host(self.n) if SHARE_GPU else NS.NativeComm.nccl(self.n)
            self.native = {"comm": comm, "NS": NS, "A": self.sp.matrix, "b": b,
                           "theta": torch.zeros_like(b) if cfg != "c5" else None}
            self.spec = P.CompositeSpec((2, 3, 4, 5))
            self.plan8 = P.table_plans()[8][0]
            self.plan16 = P.plan_order(16)
            self.mmm_per_step = 18
            if cfg == "c5":
                st = P.initial_richardson(self.sp, b, 0, 1, order=16, q=16)
                inner = st.inner
                self.native["state"] = [comm.rows_of(m) for m in (
                    inner.estimate, inner.residual, inner.accel_estimate,
                    inner.accel_residual)] + [None, None]
                self.native["theta"] = st.theta
                del st, inner
                # the recursive steps only read A: drop S^-1 and B (2 x 8.6 GB at n=32768)
                self.sp = P.Splitting(precond=self.sp.matrix[:1, :1],
                                      residual=self.sp.matrix[:1, :1], matrix=self.sp.matrix,
                                      kind="scalar", verify=False)
                del a
                self.a = None
            else:
                st = P.initial_series(self.sp, 0, 1, order={"c4": 2, "c3": 8}[cfg])
                self.native["g"] = comm.rows_of(st.estimate)
                self.native["f"] = comm.rows_of(st.residual)
                del st
            self.sharded = {"comm": comm, "native": True}
            torch.cuda.empty_cache()
            if cfg == "c5":
                self.step()  # first recursive call builds the carried weight (untimed)
            return
        if self.world > 1 and cfg in ("c4", "c3"):
            # block-row sharding over the ranks (sharded.py): A, S^-1, B replicated,
            # G / F row blocks, one row-panel exchange per product with a sharded
            # right operand (peer.py: copy engines + panel-gated DMMA products)
            from paper_2008_11480_b200.sharded import ShardedEngine

            comm = make_comm(self.n, self.comm_kind)
            eng = ShardedEngine(comm)
            st = P.initial_series(self.sp, 0, 1, order={"c4": 2, "c3": 8}[cfg])
            self.sharded = {
                "eng": eng, "comm": comm,
                "A": eng.replicated(self.sp.matrix), "P": eng.replicated(self.sp.precond),
                "B": eng.replicated(self.sp.residual), "b": eng.replicated(b),
                "g": eng.local(st.estimate[comm.r0:comm.r1].clone()),
                "f": eng.local(st.residual[comm.r0:comm.r1].clone()),
                "theta": eng.replicated(torch.zeros_like(b)),
            }
            del st
            self.spec = P.CompositeSpec((2, 3, 4, 5))
            self.plan8 = P.table_plans()[8][0]
            return
        if cfg == "c5":
            self.st = P.initial_richardson(self.sp, b, 0, 1, order=16, q=16)
            # the recursive steps only read A: drop S^-1, B and the unsymmetrised A
            # (3 x 8.6 GB at n=32768) before the 6-matrix state starts double-buffering
            self.sp = P.Splitting(precond=self.sp.matrix[:1, :1], residual=self.sp.matrix[:1, :1],
                                  matrix=self.sp.matrix, kind="scalar", verify=False)
            del a
            self.a = None
            torch.cuda.empty_cache()
            self.plan16 = P.plan_order(16)
            self.mmm_per_step = 18
            if self.world > 1:
                # block-row sharded recursive step (sharded.py) from the same initial state
                from paper_2008_11480_b200.sharded import ShardedEngine

                comm = make_comm(self.n, self.comm_kind)
                eng = ShardedEngine(comm)
                rows = slice(comm.r0, comm.r1)
                inner = self.st.inner
                self.sharded = {
                    "eng": eng, "comm": comm, "A": eng.replicated(self.sp.matrix),
                    "b": eng.replicated(b), "theta": eng.replicated(self.st.theta),
                    "state": [eng.local(m[rows].clone()) for m in
                              (inner.estimate, inner.residual, inner.accel_estimate,
                               inner.accel_residual)] + [None, None],
                }
                self.st = None
                torch.cuda.empty_cache()
                self.workload += f" [block-row x{self.world}]"
                self.step()  # first recursive call builds the carried weight (untimed)
                return
            self.st = P.richardson_recursive_step(self.st, self.sp.matrix, b,
                                                  factor_plan=self.plan16, doubling_sum=True)
        else:
            order = {"c4": 2, "c3": 8, "c1": 3}[cfg]
            self.st = P.initial_series(self.sp, 0, 1, order=order)
            self.theta = torch.zeros_like(b)
        self.spec = P.CompositeSpec((2, 3, 4, 5))
        self.plan8 = P.table_plans()[8][0]
        self.parts = None
        if cfg == "c4" and self.hoist:
            # opt-in, labelled: T_comp / R_comp evaluated once (19 products, untimed setup)
            self.parts = P.composite_parts(self.sp.matrix, self.sp, self.spec, P.MulCounter())
            self.workload = self.workload.replace("composite NS", "composite NS [HOISTED parts, 3 products/step]")

    def step(self):
        P = self.P
        cfg = self.cfg
        if getattr(self, "native", None) is not None:
            s = self.native
            NS, comm = s["NS"], s["comm"]
            if cfg == "c5":
                s["state"], s["theta"] = NS.richardson_recursive_step(
                    comm, s["state"], s["A"], s["theta"], s["b"], 16, factor_plan=self.plan16,
                    doubling_sum=True)
                return
            s["theta"] = NS.plain_richardson(comm, s["theta"], s["g"], s["A"], s["b"])
            if cfg == "c4":
                s["g"], s["f"] = NS.composite_step(comm, s["g"], s["f"], s["A"], self.sp.precond,
                                                   self.sp.residual, self.sp.matrix,
                                                   (2, 3, 4, 5), 2)
            else:
                s["g"], s["f"] = NS.ns_step(comm, s["g"], s["f"], s["A"], 8, self.plan8)
            return
        if cfg == "c2":
            self.p2, self.f2, self.t2 = P.batched_composite_richardson(
                self.a2, self.b2, self.pre2, self.res2, self.pre2, self.res2, self.t2 * 0, (2, 3),
                2, self.iters_per_step)
            return
        if cfg == "c1":
            s = self.c1
            s["p_out"], s["f_out"], s["t_out"] = P.batched_ns_richardson(
                s["a"], s["b"], s["p"], s["f"], s["t"], 3, self.iters_per_step)
            return
        if cfg == "c5":
            if self.sharded is not None:
                s = self.sharded
                g, f, l, r, om, ns = s["state"]
                g, f, l, r, om, ns, s["theta"] = s["eng"].richardson_recursive_step(
                    g, f, l, r, om, ns, s["A"], s["theta"], s["b"], 16, factor_plan=self.plan16,
                    doubling_sum=True)
                s["state"] = [g, f, l, r, om, ns]
                return
            self.st = P.richardson_recursive_step(self.st, self.sp.matrix, self.b,
                                                  factor_plan=self.plan16, doubling_sum=True)
            return
        if self.sharded is not None and "gc" in self.sharded:
            s = self.sharded
            gc = s["gc"]
            s["theta"] = gc.plain_richardson(s["theta"], s["g"], s["A"], s["b"])
            s["g"], s["f"] = gc.step(s["g"], s["f"], s["A"], s["P"], s["B"])
            return
        if self.sharded is not None:
            s = self.sharded
            eng = s["eng"]
            s["theta"] = eng.plain_richardson(s["theta"], s["g"], s["A"], s["b"])
            if cfg == "c4":
                s["g"], s["f"] = eng.composite_step(s["g"], s["f"], s["A"], s["P"], s["B"],
                                                    (2, 3, 4, 5), 2)
            else:
                s["g"], s["f"] = eng.ns_step(s["g"], s["f"], s["A"], 8, plan=self.plan8)
            return
        self.theta = P.plain_richardson(self.theta, self.st.estimate, self.sp.matrix, self.b, self.st.ctr)
        if cfg == "c4":
            self.st = P.composite_step(self.st, self.sp.matrix, self.sp, self.spec, 2,
                                       executor=self.executor, parts=self.parts)
        elif cfg == "c3":
            self.st = P.ns_step(self.st, self.sp.matrix, plan=self.plan8)
        else:
            self.st = P.ns_step(self.st, self.sp.matrix)

    def e2e_outputs_match(self, host) -> bool:
        """The outputs an e2e step left in ``host["out"]`` against the device-resident
        step from the same state (c4 / c3): bitwise, since the gated / row-block
        step computes the same products in the same order.  Untimed."""
        import torch

        P = self.P
        if self.cfg in ("c1", "c2"):  # the resident run from the state the host copies hold
            if self.cfg == "c1":
                s = self.c1
                outs = P.batched_ns_richardson(s["a"], s["b"], s["p"], s["f"], s["t"], 3,
                                               self.iters_per_step)
                back = host["pack_out"].to("cuda")
                nm = s["p"].numel()
                got = (back[:nm], back[nm:2 * nm], back[2 * nm:])
            else:
                outs = P.batched_composite_richardson(
                    self.a2, self.b2, self.pre2, self.res2, self.p2, self.f2, self.t2, (2, 3), 2,
                    self.iters_per_step)
                got = tuple(host["out"][k].to("cuda") for k in ("p", "f", "t"))
            ok = True
            for key, dev, g in zip(("p", "f", "t"), outs, got):
                if not torch.equal(g.reshape(dev.shape), dev):
                    ok = False
                    print(f"bench: e2e output {key!r} differs from the device-resident run: "
                          f"max |diff| {(g.reshape(dev.shape) - dev).abs().max().item():.3e}",
                          file=sys.stderr)
            return ok
        if self.cfg == "c4":
            ref = P.composite_step(self.st, self.sp.matrix, self.sp, self.spec, 2,
                                   executor=self.executor)
        else:
            ref = P.ns_step(self.st, self.sp.matrix, plan=self.plan8)
        theta = P.plain_richardson(self.theta, self.st.estimate, self.sp.matrix, self.b,
                                   P.MulCounter())
        ok = True
        for key, dev in (("g", ref.estimate), ("f", ref.residual), ("theta", theta)):
            back = host["out"][key].to(dev.device, non_blocking=True).reshape(dev.shape)
            if not torch.equal(back, dev):
                ok = False
                print(f"bench: e2e output {key!r} differs from the device-resident step: "
                      f"max |diff| {(back - dev).abs().max().item():.3e}", file=sys.stderr)
            del back
        return ok

    def e2e_step(self, host):
        """The public API called with HOST inputs: H2D of the step's inputs from pinned
        memory, the step, D2H of its result; returns (h2d_bytes, d2h_bytes)."""
        if self.cfg not in ("c4", "c3"):
            raise ValueError("e2e is measured for the dense configs c3 / c4")
        return self._e2e_step_overlapped(host)

    def _e2e_step_overlapped(self, host):
        """c4 / c3 through the public API with HOST inputs, copies overlapped with the
        step: the inputs are copied H2D in row panels on a copy stream, each
        panel raising a flag, and the step (``input_panels=...``) gates its DMMA
        loads per panel, so the first product starts once the first panels are
        in (not after whole matrices); G' is read back while F' = I - G' A is
        computed and F' row block by row block (``residual_chunks``).  The
        plain-Richardson products run while F' goes back."""
        import torch

        from paper_2008_11480_b200 import _lib

        P = self.P
        dev = self.a.device
        main = torch.cuda.current_stream(dev)
        if not hasattr(self, "_copy_streams"):
            self._copy_streams = (torch.cuda.Stream(dev), torch.cuda.Stream(dev))
            self._e2e_flags = torch.zeros(96, dtype=torch.int32, device=dev)
            self._e2e_epoch = 0
        up, down = self._copy_streams
        up.wait_stream(main)
        d, ev = {}, {}
        n = self.n
        # row panels of the inputs = row blocks of G' / F'; at least 1024 rows each,
        # so every block product stays on the emulated backend (its min_dim)
        npanels = int(os.environ.get("SI_BENCH_E2E_PANELS", "0")) or max(1, min(8, n // 1024))
        bounds = [n * p // npanels for p in range(npanels + 1)]
        h = _lib.handle(dev.index)
        self._e2e_epoch += 1
        epoch = self._e2e_epoch
        flags = self._e2e_flags
        slot = {"a": (0, 5), "g": (1,), "f": (2,), "precond": (3,), "residual": (4,)}

        def panel(k, p):
            r0, r1 = bounds[p], bounds[p + 1]
            d[k][r0:r1].copy_(host["in"][k][r0:r1], non_blocking=True)
            for i in slot[k]:
                _lib.call("si_stream_write_u32", h, flags.data_ptr() + 4 * (16 * i + p), epoch,
                          up.cuda_stream)

        if self.cfg == "c4":
            # the first product B S^-1 + S^-1 needs B's first row tiles and all of
            # S^-1's k-panels: B panel 0, S^-1, the rest of B, then A, G, F
            order = ("precond", "residual", "a", "g", "f", "b", "theta")
            first_a, first_b, rest = "residual", "precond", ("a", "g", "f")
        else:
            # the first product F G + G (h8 plan): F's first rows, all of G, then
            # the rest of F and A
            order = ("g", "f", "a", "b", "theta")
            first_a, first_b, rest = "f", "g", ("a",)
        with torch.cuda.stream(up):
            for k in order:
                d[k] = torch.empty(host["in"][k].shape, dtype=torch.float64, device=dev)
                d[k].record_stream(main)
            panel(first_a, 0)
            for p in range(npanels):
                panel(first_b, p)
            ev[first_b] = torch.cuda.Event()
            ev[first_b].record(up)
            for p in range(1, npanels):
                panel(first_a, p)
            ev[first_a] = torch.cuda.Event()
            ev[first_a].record(up)
            for k in rest:
                for p in range(npanels):
                    panel(k, p)
                ev[k] = torch.cuda.Event()
                ev[k].record(up)
            for k in ("b", "theta"):
                d[k].copy_(host["in"][k], non_blocking=True)
                ev[k] = torch.cuda.Event()
                ev[k].record(up)
        st = P.NsState(estimate=d["g"], residual=d["f"], step=0, order=self.st.order,
                       series_order=1, ctr=P.MulCounter())
        g_done = torch.cuda.Event()
        chunks = [torch.cuda.Event() for _ in range(npanels)]
        if self.cfg == "c4":
            sp = P.Splitting(precond=d["precond"], residual=d["residual"], matrix=d["a"],
                             kind="scalar", verify=False)
            new = P.composite_step(st, sp.matrix, sp, self.spec, 2, executor=self.executor,
                                   input_panels=(flags, epoch, npanels), residual_chunks=chunks,
                                   estimate_done=g_done)
        else:
            new = P.ns_step(st, d["a"], plan=self.plan8, input_panels=(flags, epoch, npanels),
                            residual_chunks=chunks, estimate_done=g_done)
        interleaved = self.cfg == "c4"  # composite_step: G' and F' final per row block
        with torch.cuda.stream(down):
            new.estimate.record_stream(down)
            new.residual.record_stream(down)
        if not interleaved:
            down.wait_event(g_done)
            with torch.cuda.stream(down):
                host["out"]["g"].copy_(new.estimate, non_blocking=True)
        if chunks:  # row block by row block, while the next blocks are computed
            for p, e in enumerate(chunks):
                down.wait_event(e)
                with torch.cuda.stream(down):
                    r0, r1 = bounds[p], bounds[p + 1]
                    if interleaved:
                        host["out"]["g"][r0:r1].copy_(new.estimate[r0:r1], non_blocking=True)
                    host["out"]["f"][r0:r1].copy_(new.residual[r0:r1], non_blocking=True)
        else:
            f_done = torch.cuda.Event()
            f_done.record(main)
            down.wait_event(f_done)
            with torch.cuda.stream(down):
                host["out"]["f"].copy_(new.residual, non_blocking=True)
        for k in ("a", "g", "b", "theta"):
            main.wait_event(ev[k])
        theta = P.plain_richardson(d["theta"], st.estimate, d["a"], d["b"], st.ctr)
        host["out"]["theta"].copy_(theta, non_blocking=True)
        main.wait_stream(down)
        h2d = sum(host["in"][k].numel() * 8 for k in order)
        d2h = sum(v.numel() * 8 for v in host["out"].values())
        return h2d, d2h

    def pinned_inputs_resident(self):
        """Host (pinned) inputs and outputs of one resident-kernel launch (c1 / c2)."""
        import torch

        def pin(t):
            h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
            h.copy_(t)
            return h

        if self.cfg == "c1":
            # one system: the inputs travel as one packed pinned buffer (one copy
            # each way instead of five / three small ones)
            s = self.c1
            host = {"in": {k: pin(s[k]) for k in ("a", "b", "p", "f", "t")}}
            host["pack_in"] = pin(torch.cat([s[k].reshape(-1) for k in ("a", "b", "p", "f", "t")]))
            host["pack_out"] = torch.empty(2 * s["p"].numel() + s["t"].numel(),
                                           dtype=torch.float64, pin_memory=True)
        else:
            host = {"in": {"a": pin(self.a2), "b": pin(self.b2), "pre": pin(self.pre2),
                           "res": pin(self.res2), "p": pin(self.p2), "f": pin(self.f2),
                           "t": pin(self.t2)}}
        host["out"] = {k: torch.empty_like(host["in"][k], pin_memory=True) for k in ("p", "f", "t")}
        return host

    def e2e_step_resident(self, host):
        """One resident run through the public API from host buffers.  c2: one
        launch fed by chunks of systems (``input_chunks`` flags behind each
        chunk's copy) whose outputs go back chunk by chunk (``chunk_done``
        counters); c1: one system, one packed copy each way."""
        import torch

        P = self.P
        main = torch.cuda.current_stream()
        if not hasattr(self, "_copy_streams"):
            self._copy_streams = (torch.cuda.Stream(), torch.cuda.Stream())
        up, down = self._copy_streams
        up.wait_stream(main)
        hin, hout = host["in"], host["out"]
        if self.cfg == "c1":
            dev = host["pack_in"].to("cuda", non_blocking=True)
            d, off = {}, 0
            for k in ("a", "b", "p", "f", "t"):
                m = hin[k].numel()
                d[k] = dev[off:off + m].view(hin[k].shape)
                off += m
            # outputs written straight into one packed device buffer: one read-back
            nm, nt = hin["p"].numel(), hin["t"].numel()
            packed = torch.empty(2 * nm + nt, dtype=torch.float64, device="cuda")
            P.batched_ns_richardson(d["a"], d["b"], d["p"], d["f"], d["t"], 3,
                                    self.iters_per_step,
                                    out=(packed[:nm], packed[nm:2 * nm], packed[2 * nm:]))
            host["pack_out"].copy_(packed, non_blocking=True)
            main.wait_stream(down)
            return host["pack_in"].numel() * 8, host["pack_out"].numel() * 8
        else:
            # the batch arrives by chunks of one launch round (grid = 4 CTAs x
            # 148 SMs): the kernel waits per chunk for its flag, counts finished
            # systems per chunk, and each chunk's outputs go back as soon as
            # its counter is full
            from paper_2008_11480_b200 import _lib

            batch = hin["a"].shape[0]
            chunk = 4 * torch.cuda.get_device_properties(0).multi_processor_count
            nchunks = (batch + chunk - 1) // chunk
            if not hasattr(self, "_c2_flags") or self._c2_flags.numel() < nchunks:
                self._c2_flags = torch.zeros(nchunks, dtype=torch.int32, device="cuda")
                self._c2_done = torch.zeros(nchunks, dtype=torch.int32, device="cuda")
                self._c2_target = [0] * nchunks
                self._c2_epoch = 0
            self._c2_epoch += 1
            epoch = self._c2_epoch
            h = _lib.handle(0)
            d = {}
            with torch.cuda.stream(up):
                for k, v in hin.items():
                    d[k] = torch.empty(v.shape, dtype=v.dtype, device="cuda")
                    d[k].record_stream(main)
                for c in range(nchunks):
                    lo, hi = c * chunk, min(batch, (c + 1) * chunk)
                    for k, v in hin.items():
                        d[k][lo:hi].copy_(v[lo:hi], non_blocking=True)
                    _lib.call("si_stream_write_u32", h, self._c2_flags.data_ptr() + 4 * c, epoch,
                              up.cuda_stream)
            # the read-back must not wait for the whole launch: only for main's work
            # before it (the output blocks are handed out from memory freed by
            # that work); each chunk then waits on its own counter
            before = torch.cuda.Event()
            before.record(main)
            p, f, t = P.batched_composite_richardson(
                d["a"], d["b"], d["pre"], d["res"], d["p"], d["f"], d["t"], (2, 3), 2,
                self.iters_per_step, input_chunks=(self._c2_flags, epoch, chunk),
                chunk_done=self._c2_done)
            down.wait_event(before)
            with torch.cuda.stream(down):
                for c in range(nchunks):
                    lo, hi = c * chunk, min(batch, (c + 1) * chunk)
                    self._c2_target[c] += hi - lo
                    _lib.call("si_stream_wait_u32", h, self._c2_done.data_ptr() + 4 * c,
                              self._c2_target[c], down.cuda_stream)
                    for k, v in (("p", p), ("f", f), ("t", t)):
                        hout[k][lo:hi].copy_(v[lo:hi], non_blocking=True)
                for v in (p, f, t):
                    v.record_stream(down)
            main.wait_stream(down)
        h2d = sum(v.numel() * 8 for v in hin.values())
        d2h = sum(v.numel() * 8 for v in hout.values())
        return h2d, d2h

    def pinned_inputs_sharded(self):
        """This rank's host inputs of a sharded step: the replicated operands and
        its G / F row blocks, in pinned memory; outputs likewise."""
        import torch

        s = self.sharded
        eng = s["eng"]

        def pin(t):
            h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
            h.copy_(t)
            return h

        host = {"in": {"a": pin(s["A"].t), "precond": pin(s["P"].t), "residual": pin(s["B"].t),
                       "b": pin(s["b"].t), "theta": pin(s["theta"].t),
                       "g": pin(eng.rows_of(s["g"])), "f": pin(eng.rows_of(s["f"]))}}
        host["out"] = {k: torch.empty_like(host["in"][k], pin_memory=True)
                       for k in ("g", "f", "theta")}
        return host

    def e2e_step_sharded(self, host):
        """One sharded step through the block-row API from host buffers: H2D of this
        rank's inputs, the step, D2H of its G' / F' row blocks and theta'."""
        s = self.sharded
        eng = s["eng"]
        dev = s["A"].t.device
        d = {k: v.to(dev, non_blocking=True) for k, v in host["in"].items()}
        A, Pm, B = eng.replicated(d["a"]), eng.replicated(d["precond"]), eng.replicated(d["residual"])
        theta = eng.plain_richardson(eng.replicated(d["theta"]), eng.local(d["g"]), A,
                                     eng.replicated(d["b"]))
        if "gc" in s:  # composite parts on GPU groups (grouped.py)
            g, f = s["gc"].step(eng.local(d["g"]), eng.local(d["f"]), A, Pm, B)
        elif self.cfg == "c4":
            g, f = eng.composite_step(eng.local(d["g"]), eng.local(d["f"]), A, Pm, B,
                                      (2, 3, 4, 5), 2)
        else:
            g, f = eng.ns_step(eng.local(d["g"]), eng.local(d["f"]), A, 8, plan=self.plan8)
        host["out"]["g"].copy_(eng.rows_of(g), non_blocking=True)
        host["out"]["f"].copy_(eng.rows_of(f), non_blocking=True)
        host["out"]["theta"].copy_(theta.t, non_blocking=True)
        h2d = sum(v.numel() * 8 for v in host["in"].values())
        d2h = sum(v.numel() * 8 for v in host["out"].values())
        return h2d, d2h

    def pinned_inputs_c5(self):
        """c5: the numpy-facing call's inputs (A, b, theta and the six carried
        state matrices) and outputs in pinned host memory; the device copy of
        the state is released (the GPU holds one state at a time: 8.6 GB per
        matrix)."""
        import torch

        def pin(t):
            h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
            h.copy_(t)
            return h

        st = self.st
        inner = st.inner
        host = {"in": {"a": pin(self.sp.matrix), "b": pin(self.b), "theta": pin(st.theta),
                       "g": pin(inner.estimate), "f": pin(inner.residual),
                       "l": pin(inner.accel_estimate), "r": pin(inner.accel_residual),
                       "omega": pin(st.omega), "ns": pin(st.ns_part)}}
        host["out"] = {k: torch.empty_like(host["in"][k], pin_memory=True)
                       for k in ("theta", "g", "f", "l", "r", "omega", "ns")}
        self.st = None
        self.sp = None
        self.b = None
        torch.cuda.empty_cache()
        return host

    def e2e_step_c5(self, host):
        """One steady-state recursive step (factorised order 16, the bench DAG)
        through the public API from host buffers, copies overlapped with the
        step: the inputs go H2D on a copy stream in the order the DAG first
        reads them (R for the power sum, L, A, omega, N, b, theta; G and F,
        which the steady-state DAG does not read, last), each behind an event
        the step waits on right before that input's first use; every field of
        the new state goes D2H on a second copy stream as soon as the step
        records it final (L', R', G', F', N', omega', theta')."""
        import torch

        P = self.P
        dev = torch.device("cuda", torch.cuda.current_device())
        main = torch.cuda.current_stream(dev)
        if not hasattr(self, "_copy_streams"):
            self._copy_streams = (torch.cuda.Stream(dev), torch.cuda.Stream(dev))
        up, down = self._copy_streams
        names = {"a": "a", "b": "b", "theta": "theta", "g": "estimate", "f": "residual",
                 "l": "accel_estimate", "r": "accel_residual", "omega": "omega", "ns": "ns_part"}
        order = ("r", "l", "a", "omega", "ns", "b", "theta", "g", "f")
        # buffers from the step's own (main-stream) pool, as the unoverlapped
        # call had them: at n = 32768 the step runs at the edge of the 180 GB
        d = {k: torch.empty(host["in"][k].shape, dtype=torch.float64, device=dev) for k in order}
        up.wait_stream(main)
        ready = {}
        with torch.cuda.stream(up):
            for k in order:
                d[k].record_stream(up)
                d[k].copy_(host["in"][k], non_blocking=True)
                ready[names[k]] = torch.cuda.Event()
                ready[names[k]].record(up)
        inner = P.DoubleNsState(estimate=d["g"], residual=d["f"], accel_estimate=d["l"],
                                accel_residual=d["r"], step=1, order=16, series_order=1,
                                ctr=P.MulCounter())
        st = P.RichardsonState(theta=d["theta"], inner=inner, q=16, omega=d["omega"],
                               ns_part=d["ns"], step=1, ctr=inner.ctr)
        a, b = d.pop("a"), d.pop("b")
        del d
        outs = ("accel_estimate", "accel_residual", "estimate", "residual", "ns_part", "omega",
                "theta")
        done = {k: torch.cuda.Event() for k in outs}
        new = P.richardson_recursive_step(st, a, b, factor_plan=self.plan16, doubling_sum=True,
                                          inputs_ready=ready, outputs_done=done)
        del st, inner
        out = host["out"]
        fields = {"accel_estimate": ("l", new.inner.accel_estimate),
                  "accel_residual": ("r", new.inner.accel_residual),
                  "estimate": ("g", new.inner.estimate), "residual": ("f", new.inner.residual),
                  "ns_part": ("ns", new.ns_part), "omega": ("omega", new.omega),
                  "theta": ("theta", new.theta)}
        for k in outs:  # the order the step finishes them in
            hk, v = fields[k]
            down.wait_event(done[k])
            v.record_stream(down)
            with torch.cuda.stream(down):
                out[hk].copy_(v, non_blocking=True)
        main.wait_stream(down)
        h2d = sum(v.numel() * 8 for v in host["in"].values())
        d2h = sum(v.numel() * 8 for v in out.values())
        return h2d, d2h

    def pinned_inputs(self):
        import torch

        def pin(t):
            h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
            h.copy_(t)
            return h

        host = {"in": {"a": pin(self.sp.matrix), "g": pin(self.st.estimate),
                       "f": pin(self.st.residual), "b": pin(self.b), "theta": pin(self.theta)},
                "out": {}}
        if self.cfg == "c4":  # the composite step's parts read the splitting too
            host["in"]["precond"] = pin(self.sp.precond)
            host["in"]["residual"] = pin(self.sp.residual)
        host["out"] = {"g": torch.empty_like(host["in"]["g"], pin_memory=True),
                       "f": torch.empty_like(host["in"]["f"], pin_memory=True),
                       "theta": torch.empty_like(host["in"]["theta"], pin_memory=True)}
        return host


def cpu_part_sample(n: int, a=None, precond=None, residual=None):
    """Bounded CPU sample for our arm's ``cpu_baseline`` (c4/c5, ~10-20 s): the
    rate-2 part of the composite step executed through the oracle at full n --
    T = B S^-1 + S^-1 (geometric_apply, st:432-457) and Gamma = I - T A
    (ns:206-210), two n^3 products with the reference's n^2 temporaries
    (identity, add, subtract).  Returns (seconds, products executed)."""
    import numpy as np

    from oracle import seriesinv_oracle as O

    if a is None:
        rng = np.random.default_rng(1)
        a = rng.standard_normal((n, n))
        precond = np.eye(n) / n
        residual = np.eye(n) - a / n
    ctr = O.Counter()
    O.mm(a[:256, :256], a[:256, :256], ctr)  # spin up the BLAS thread pool
    t0 = time.perf_counter()
    t = O.geometric_apply(residual, precond, 2, a, ctr)
    gamma = np.eye(n) - O.mm(t, a, ctr)
    dt = time.perf_counter() - t0
    del t, gamma
    return dt, 2


def reference_step_seconds(cfg: str, n: int, batch: int = 16384):
    """c1-c3: seconds the CPU oracle needs for ONE bench step of `cfg` (the same
    unit as our arm's step), executed on a bounded sample; returns (seconds,
    description).

    c1: the whole 30-iteration run, executed (milliseconds; best of 20 runs).
    c2: 50 iterations of 64 of the systems, executed, scaled to the full batch.
    c3: one full-size iteration (n=4096: plain Richardson + h8 ns_step), executed."""
    import numpy as np

    from oracle import seriesinv_oracle as O
    from paper_2008_11480_b200 import configs

    if cfg == "c1":
        a, b = configs.c1_dense_small(n=n)
        sp = O.split_scalar(a, O.inf_norm(a) / 2.0)
        best = float("inf")
        for _ in range(20):
            st = O.initial_series(sp, 0, 1, 3)
            th = np.zeros_like(b)
            t0 = time.perf_counter()
            for _ in range(30):
                th = O.plain_richardson(th, st.estimate, sp.matrix, b, st.ctr)
                st = O.ns_step(st, sp.matrix)
            best = min(best, time.perf_counter() - t0)
        return best, "whole 30-iteration run through the oracle (best of 20)"
    if cfg == "c2":
        k = 64
        a, b = configs.c2_batched(batch=k)
        t0 = time.perf_counter()
        for i in range(k):
            sp = O.split_scalar(a[i], O.inf_norm(a[i]) / 2.0)
            st = O.initial_series(sp, 0, 1, 2)
            th = np.zeros(a.shape[1])
            for _ in range(50):
                th = O.plain_richardson(th, st.estimate, sp.matrix, b[i], st.ctr)
                st = O.composite_step(st, sp.matrix, sp, (2, 3), 2)
        t = time.perf_counter() - t0
        return t * batch / k, f"50 iterations of {k} systems through the oracle, x{batch // k} systems"
    if cfg == "c3":
        a, b = configs.c3_gram(n=n)
        sp = O.split_scalar(a, O.inf_norm(a) / 2.0)
        st = O.initial_series(sp, 0, 1, 8)
        th = np.zeros_like(b)
        plan = O.TABLE_ROOTS[8][0][1]
        t0 = time.perf_counter()
        th = O.plain_richardson(th, st.estimate, sp.matrix, b, st.ctr)
        st = O.ns_step(st, sp.matrix, plan)
        return time.perf_counter() - t0, f"one full-size iteration (n={n}) through the oracle"
    raise ValueError(cfg)


def reference_executed_steps(cfg: str, n: int, max_steps: int, budget_s: float):
    """c4/c5 reference arm: FULL steps of the reference DAG executed through the
    oracle on the host cores (no extrapolation for c4).

    c4: plain Richardson (64 RHS) + composite_step((2,3,4,5), 2) at n (the
        bench workload itself; ~2 min per step on 16 cores), from the
        config's initial state.
    c5: one steady-state recursive step (richardson.py:111-189, Horner, 34
        products) at min(n, 16384) -- a full n=32768 step is ~25 min of CPU --
        on the config-5 recipe at that size, from a synthetic carried state
        (S^-1 / B standing in for G, L / F, R and for omega / N: the products
        are dense and their cost does not depend on the values); the time is
        scaled by (n / 16384)^3 and labelled.
    Steps run while the next one still fits in ``budget_s`` (at least one, at
    most ``max_steps``).  Returns (step seconds list, description)."""
    import numpy as np

    from oracle import seriesinv_oracle as O
    from paper_2008_11480_b200 import configs

    times = []
    if cfg == "c4":
        t_setup = time.perf_counter()
        a, b = configs.c4_householder(n=n, rhs=64)
        sp = O.split_scalar(a, O.inf_norm(a) / 2.0)
        del a
        st = O.initial_series(sp, 0, 1, 2)
        theta = np.zeros_like(b)
        setup = time.perf_counter() - t_setup
        O.mm(sp.matrix[:256, :256], sp.matrix[:256, :256], O.Counter())  # BLAS pool warm
        t_all = time.perf_counter()
        while True:
            t0 = time.perf_counter()
            theta = O.plain_richardson(theta, st.estimate, sp.matrix, b, st.ctr)
            st = O.composite_step(st, sp.matrix, sp, (2, 3, 4, 5), 2)
            times.append(time.perf_counter() - t0)
            spent = time.perf_counter() - t_all
            if len(times) >= max_steps or spent + times[-1] > budget_s:
                break
        mmm = st.ctr.mmm // len(times)
        return times, (f"{len(times)} full step(s) executed at n={n} through the oracle "
                       f"(plain Richardson, 64 RHS + composite_step (2,3,4,5) order_n=2: "
                       f"{mmm} n^3 products + 2 n^2 r products each, the reference's n^2 "
                       f"temporaries included; inputs built on the host in {setup:.0f} s, untimed)")
    if cfg == "c5":
        sn = min(n, 16384)
        m = int(round(sn * 40000 / 32768))
        rng = np.random.default_rng(0)
        g = rng.standard_normal((m, sn))
        b = rng.standard_normal((sn, 256))
        a = g.T @ g / m + 1e-3 * np.eye(sn)
        del g
        sp = O.split_scalar(a, O.inf_norm(a) / 2.0)
        del a
        ctr = O.Counter()
        inner = O.DoubleNS(sp.precond.copy(), sp.residual.copy(), sp.precond.copy(),
                           sp.residual.copy(), 1, 16, 1, ctr)
        st = O.Rich(np.zeros_like(b), inner, 16, sp.precond.copy(), sp.precond.copy(), 1, ctr)
        O.mm(sp.matrix[:256, :256], sp.matrix[:256, :256], O.Counter())
        t_all = time.perf_counter()
        while True:
            c0 = ctr.mmm
            t0 = time.perf_counter()
            st = O.richardson_recursive_step(st, sp.matrix, b)
            times.append((time.perf_counter() - t0) * (n / sn) ** 3)
            products = ctr.mmm - c0
            spent = time.perf_counter() - t_all
            if len(times) >= max_steps or spent + times[-1] * (sn / n) ** 3 > budget_s:
                break
        scale = "" if sn == n else f", scaled by (n/{sn})^3 to n={n} (extrapolated)"
        return times, (f"{len(times)} steady-state recursive step(s) (Horner order 16, {products} "
                       f"n^3 products + 2 n^2 r products, r=256) executed at n={sn} through the "
                       f"oracle from a synthetic carried state{scale}")
    raise ValueError(cfg)


def config_obj(cfg: str, n: int, batch: int = 16384) -> dict:
    """The `config` object: identical in both arms (the parallelism / L2 /
    sampling details are top-level keys)."""
    return {"workload": workload_desc(cfg, n, batch), "n": n,
            "rhs": {"c4": 64, "c5": 256, "c2": 1, "c1": 1, "c3": 1}[cfg]}


# --------------------------------------------------------------------------- arms


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cfg = args.config
    n = args.n or {"c4": 16384, "c3": 4096, "c1": 64, "c5": 32768, "c2": 32}[cfg]
    w = Workload(cfg, n)
    w.r = {"c4": 64, "c5": 256}.get(cfg, 1)
    w.mmm_per_step = 34  # the reference's recursive step is Horner (ri:111-189)
    w.batch = (args.n or 16384) if cfg == "c2" else 16384
    if cfg == "c2":
        w.n = 32
    w.iters_per_step = {"c1": 30, "c2": 50}.get(cfg, 1)
    flops = w.flops()
    cores = use_all_host_threads()
    if cfg in ("c4", "c5"):
        # full reference steps, executed (c5: at n=16384, scaled by n^3)
        step_times, sample = reference_executed_steps(cfg, w.n, args.steps, args.ref_budget)
        steps_timed, warm = len(step_times), 0
        executed = {"executed_iterations": len(step_times), "steps_requested": args.steps,
                    "warmup_requested": args.warmup,
                    "note": ("each timed step is one full reference step; steps run while the "
                             f"next fits in --ref-budget {args.ref_budget:.0f} s, so 'steps' is "
                             "the executed count (no warm-up step: a BLAS warm-up product only)")}
    else:
        # each step: a bounded sample of one bench step of the workload (see
        # reference_step_seconds for what is executed)
        step_times, sample = [], ""
        for i in range(args.warmup + args.steps):
            s, sample = reference_step_seconds(cfg, w.n, batch=w.batch)
            if i >= args.warmup:
                step_times.append(s)
        steps_timed, warm = args.steps, args.warmup
        executed = {"executed_iterations": args.steps * w.iters_per_step}
    step_s = statistics.mean(step_times)
    value = w.iters_per_step / step_s
    sample = f"{sample}; numpy/OpenBLAS with {cores} host threads"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "iters/s",
        "n_gpus": world, "steps": steps_timed, "warmup": warm,
        "ms_per_step": step_s * 1e3, "iters_per_step": w.iters_per_step,
        "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_obj(cfg, w.n, w.batch),
        "parallelism": f"host CPU, {cores} threads (rank 0 only)",
        "tflops": flops / step_s / 1e12,
        "cpu_baseline": {"value": value, "unit": "iters/s", "cores": cores, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": "iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "step_seconds": step_times,
        **executed,
    }
    print(json.dumps(line), flush=True)
    return 0


def sharded_e2e(w, args, world, stream):
    """e2e of a sharded step: this rank's host inputs (replicated operands and
    its row blocks) copied in, the step, its row blocks copied out."""
    import torch

    host = w.pinned_inputs_sharded()
    ksteps = max(1, min(args.steps, 3))
    w.e2e_step_sharded(host)  # warm
    torch.cuda.synchronize()
    barrier(world)
    f0 = torch.cuda.Event(enable_timing=True)
    f1 = torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    for _ in range(ksteps):
        h2d, d2h = w.e2e_step_sharded(host)
    f1.record(stream)
    torch.cuda.synchronize()
    e_ms = max_over_ranks(f0.elapsed_time(f1), world)
    del host
    # one job of fixed size over all ranks; bytes are this rank's copies
    return {"value": ksteps / (e_ms / 1e3), "unit": "iters/s",
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "steps": ksteps,
            "bytes": "per rank (A, S^-1, B, b, theta replicated; G, F row blocks)"}


def our_cpu_baseline(w, flops: float) -> dict:
    """`cpu_baseline` of our arm (rank 0, N=1): the oracle on the host cores on a
    bounded sample of the same workload (10-30 s of CPU).  c1-c3: the executed
    samples of reference_step_seconds; c4/c5: the rate-2 part of the composite
    step (2 full-size products with the reference's n^2 temporaries) executed,
    scaled to the reference DAG's step by FLOPs (c5: Horner, 34 products; its
    sample at n=16384 on random matrices, scaled by n^3)."""
    cores = use_all_host_threads()
    if w.cfg in ("c1", "c2", "c3"):
        s, desc = reference_step_seconds(w.cfg, w.n, batch=getattr(w, "batch", 16384))
    else:
        if w.cfg == "c4":
            host = [t.cpu().numpy() for t in (w.sp.matrix, w.sp.precond, w.sp.residual)]
            t, k = cpu_part_sample(w.n, *host)
            del host
            ref_flops, sn = flops, w.n
        else:
            sn = min(w.n, 16384)
            t, k = cpu_part_sample(sn)
            ref_flops = 34 * 2.0 * w.n**3 + 2 * 2.0 * w.n * w.n * w.r
        s = t / (k * 2.0 * sn**3) * ref_flops
        desc = (f"rate-2 part of the composite step ({k} products of {sn}^3 with the reference's "
                f"n^2 temporaries) executed in {t:.1f} s, scaled by the reference step DAG's "
                f"FLOPs ({ref_flops:.4e}/step) -- extrapolated")
    return {"value": w.iters_per_step / s, "unit": "iters/s", "cores": cores, "kind": "port",
            "sample": f"{desc}; numpy/OpenBLAS, all host threads"}


def config_of(w) -> dict:
    """Our arm's `config`: the reference arm's object, except for the opt-in
    hoisted variant (a different DAG, labelled in its workload string)."""
    c = config_obj(w.cfg, w.n, getattr(w, "batch", 16384))
    if w.hoist:
        c["workload"] = w.workload
    return c


def layout_note(w) -> str:
    """The multi-GPU layout details appended to the workload string (e.g. the
    GPU groups of the parts mapping) go to `parallelism`, not `config`."""
    base = workload_desc(w.cfg, w.n, getattr(w, "batch", 16384))
    extra = w.workload[len(base):].strip() if w.workload.startswith(base) and not w.hoist else ""
    return f"{extra} " if extra else ""


def rank_info(w, args, world: int, rank: int, local: int) -> dict:
    """One self-describing line per rank (stderr): device, peer access to the
    other GPUs, exchange bytes pulled, NCCL ranks -- so a multi-GPU run
    verifies its own wiring."""
    import torch

    info = {"rank": rank, "local_rank": local, "world": world}
    try:
        dev = torch.cuda.current_device()
        props = torch.cuda.get_device_properties(dev)
        info["device"] = {"index": dev, "name": props.name,
                          "pci_bus_id": getattr(props, "pci_bus_id", None),
                          "uuid": str(getattr(props, "uuid", ""))}
        info["peer_access"] = {j: torch.cuda.can_device_access_peer(dev, j)
                               for j in range(torch.cuda.device_count()) if j != dev}
    except RuntimeError as exc:
        info["device"] = f"unavailable: {exc}"
    s = w.sharded or {}
    comm = s.get("comm")
    if comm is not None:
        info["comm"] = type(comm).__name__
        if s.get("native"):
            info["gathers"], info["bytes_pulled"] = comm.stats()
        else:
            info["bytes_pulled"] = getattr(comm, "bytes_gathered", None)
            info["gathers"] = getattr(comm, "seq", None)
    if world > 1:
        import torch.distributed as dist

        info["backend"] = dist.get_backend()
        info["nccl_nranks"] = dist.get_world_size() if dist.get_backend() == "nccl" else 0
    info["share_gpu"] = SHARE_GPU
    return info


def run_ours(args):
    import torch

    world, rank, local = dist_setup(args)
    from paper_2008_11480_b200 import _lib

    w = Workload(args.config, args.n, world, hoist=args.hoist, comm=args.comm, shard=args.shard)
    w.setup()
    flops = w.flops()
    h = _lib.handle()
    if args.streams and w.cfg == "c4":
        w.executor = "streams"  # any non-None executor: parts on the library's side streams
    ozaki = args.gemm in ("ozaki", "auto") and w.cfg in ("c3", "c4", "c5")
    if ozaki:
        # after setup (the PD check / verification products stay on DMMA)
        w.P.set_gemm_backend("ozaki", moduli=args.moduli, min_dim=1024)
        w.P.set_ozaki_kernel(args.i8_kernel)
        w.i8_kernel = args.i8_kernel
    # roofline denominators, probed before any timed work (a GPU held at its
    # power cap by a long INT8 run reads far lower)
    import ctypes

    peak = ctypes.c_double()
    _lib.call("si_dmma_peak", h, 20000, ctypes.byref(peak))
    i8_peak = int8_peak_tops() if ozaki else None
    for _ in range(args.warmup):
        w.step()
    torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()

    sampler = ClockSampler(local)
    sampler.start()
    _lib.call("si_profile_begin", h)
    stream = torch.cuda.current_stream()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        w.step()
    e1.record(stream)
    torch.cuda.synchronize()
    import ctypes

    g_ms, g_fl = ctypes.c_double(), ctypes.c_double()
    g_n, launches = ctypes.c_int64(), ctypes.c_int64()
    _lib.call("si_profile_end", h, ctypes.byref(g_ms), ctypes.byref(g_fl), ctypes.byref(g_n),
              ctypes.byref(launches))
    i8_ms, i8_ops, i8_n = ctypes.c_double(), ctypes.c_double(), ctypes.c_int64()
    _lib.call("si_profile_i8", h, ctypes.byref(i8_ms), ctypes.byref(i8_ops), ctypes.byref(i8_n))
    clocks = sampler.stop()
    print("rank-info " + json.dumps(rank_info(w, args, world, rank, local)), file=sys.stderr,
          flush=True)
    barrier(world)
    ms = e0.elapsed_time(e1)
    ms_max = max_over_ranks(ms, world)
    step_s = ms_max / 1e3 / args.steps
    # sharded (c3/c4 at N > 1): every rank works on the same job -> strong scaling;
    # otherwise N independent replicas each complete `steps` iterations -> weak
    # sharded (c3/c4/c5) or batch-split (c2) at N > 1: all ranks work on ONE job of
    # fixed size -> strong scaling; otherwise N replicas each run the job -> weak
    strong = w.sharded is not None or w.split_batch
    value = (1 if strong else world) * args.steps * w.iters_per_step / (ms_max / 1e3)
    tflops = (1 if strong else world) * flops / step_s / 1e12

    achieved = (g_fl.value / (g_ms.value / 1e3) / 1e12) if g_ms.value > 0 else None

    fp64_dmma = None
    side_run = ozaki and world == 1 and not args.no_dmma_side
    if side_run and w.cfg == "c5":  # c5's e2e releases the device state: side run first
        fp64_dmma = dmma_side_run(w, args, h, flops, peak.value)
    e2e = None
    if w.sharded is not None and w.sharded.get("native"):
        e2e = {"unavailable": "--comm native: e2e is measured on the peer / nccl paths"}
    elif not args.no_e2e and args.config in ("c4", "c3") and w.sharded is not None:
        try:
            e2e = sharded_e2e(w, args, world, stream)
        except (RuntimeError, MemoryError) as exc:  # e.g. pinned host memory exhausted
            e2e = {"unavailable": f"sharded e2e failed: {exc}"[:200]}
    if not args.no_e2e and args.config in ("c1", "c2") and not w.split_batch:
        host = w.pinned_inputs_resident()
        # ~0.3-0.5 s of e2e runs (a c1 run is ~0.2 ms, a c2 run ~18 ms), at most --steps
        ksteps = max(1, min(args.steps, 2000 if args.config == "c1" else 30))
        w.e2e_step_resident(host)  # warm
        torch.cuda.synchronize()
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(ksteps):
            h2d, d2h = w.e2e_step_resident(host)
        f1.record(stream)
        torch.cuda.synchronize()
        e_ms = max_over_ranks(f0.elapsed_time(f1), world)
        e2e = {"value": world * ksteps * w.iters_per_step / (e_ms / 1e3), "unit": "iters/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "steps": ksteps}
        if w.e2e_outputs_match(host):
            e2e["outputs"] = "bitwise equal to the device-resident run from the same state"
        else:
            e2e = {"invalid": "e2e outputs differ from the device-resident run", **e2e}
            e2e["value"] = None
        torch.cuda.synchronize()
        del host
    if not args.no_e2e and args.config in ("c4", "c3") and w.sharded is None and not args.hoist:
        host = w.pinned_inputs()
        h2d = d2h = 0
        # at least ~1 s of e2e steps (3 for c4; ~100 for c3), at most --steps
        ksteps = max(1, min(args.steps, max(3, int(1.0 / max(step_s, 1e-3)))))
        w.e2e_step(host)  # warm
        torch.cuda.synchronize()
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(ksteps):
            h2d, d2h = w.e2e_step(host)
        f1.record(stream)
        torch.cuda.synchronize()
        e_ms = max_over_ranks(f0.elapsed_time(f1), world)
        e2e = {"value": world * ksteps / (e_ms / 1e3), "unit": "iters/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "steps": ksteps}
        # what the last timed e2e step read back is the device-resident step's
        # result (every step starts from the same host state)
        if w.e2e_outputs_match(host):
            e2e["outputs"] = "bitwise equal to the device-resident step from the same state"
        else:
            print("bench: the e2e step's outputs differ from the device-resident step", file=sys.stderr)
            e2e = {"invalid": "e2e outputs differ from the device-resident step", **e2e}
            e2e["value"] = None
        torch.cuda.synchronize()
        del host

    if not args.no_e2e and args.config == "c5" and w.sharded is None:
        try:
            # checksums of the device-resident step from the state the e2e step will
            # start from (the state itself is released for the host copies)
            def sums(t):
                return (t.sum().item(), t.abs().max().item())

            ref = w.P.richardson_recursive_step(w.st, w.sp.matrix, w.b, factor_plan=w.plan16,
                                                doubling_sum=True)
            want = {"theta": sums(ref.theta), "g": sums(ref.inner.estimate),
                    "f": sums(ref.inner.residual), "l": sums(ref.inner.accel_estimate),
                    "r": sums(ref.inner.accel_residual), "omega": sums(ref.omega),
                    "ns": sums(ref.ns_part)}
            del ref
            host = w.pinned_inputs_c5()
            f0 = torch.cuda.Event(enable_timing=True)
            f1 = torch.cuda.Event(enable_timing=True)
            f0.record(stream)
            h2d, d2h = w.e2e_step_c5(host)  # one step: ~37 s
            f1.record(stream)
            torch.cuda.synchronize()
            e_ms = max_over_ranks(f0.elapsed_time(f1), world)
            e2e = {"value": world / (e_ms / 1e3), "unit": "iters/s",
                   "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "steps": 1,
                   "note": "A, b, theta and the six carried n x n matrices in, the new state "
                           "and theta out; copies overlapped with the step per input / "
                           "output (si_richardson_recursive_step_ex)"}
            torch.cuda.empty_cache()
            bad = []
            for k, v in host["out"].items():  # one matrix at a time back on the device
                got = sums(v.to("cuda"))
                if got != want[k]:
                    bad.append(k)
            if bad:
                print(f"bench: c5 e2e outputs {bad} differ from the device-resident step",
                      file=sys.stderr)
                e2e = {"invalid": f"e2e outputs {bad} differ from the device-resident step",
                       **e2e}
                e2e["value"] = None
            else:
                e2e["outputs"] = ("sum and max |.| of every output equal those of the "
                                  "device-resident step from the same state")
            del host
        except (RuntimeError, MemoryError) as exc:  # pinned host memory exhausted, ...
            e2e = {"unavailable": f"c5 e2e failed: {exc}"[:200]}
        # (the device state was released for the e2e copies: c5 ends here)

    if side_run and w.cfg != "c5":  # after the e2e steps (their timing sees no DMMA-run state)
        fp64_dmma = dmma_side_run(w, args, h, flops, peak.value)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu and not args.hoist:
        cpu = our_cpu_baseline(w, flops)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "iters/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_s * 1e3,
            "iters_per_step": w.iters_per_step,
            "higher_is_better": True, "scaling": "strong" if strong else "weak",
            "vs_baseline": None,
            "dtype": (f"int8 tensor cores -> f64 (Ozaki-II FP64 emulation, {args.moduli} moduli)"
                      if ozaki else "f64"),
            "gemm_backend": "ozaki" if ozaki else "dmma",
            "parts_on_streams": w.executor is not None,
            "data": "synthetic (seeded PCG64 draws, SURVEY Appendix A recipe)",
            "config": config_of(w),
            "parallelism": layout_note(w) + (f"composite parts on GPU groups x{world} (NCCL p2p tree)"
                            if w.sharded is not None and "gc" in w.sharded
                            else f"block-row x{world} ({_COMM_LABEL['nccl' if COMM_FALLBACK else args.comm]})"
                            if w.sharded is not None
                            else f"batch split x{world} (no communication)" if w.split_batch
                            else (f"replicas x{world}" if world > 1 else "single-gpu")),
            "l2": l2_note(w),
            "tflops": tflops,
            "tflops_frac_of_dmma_peak": tflops / (world * peak.value),
            "roofline": resident_roofline(w, tflops / world, step_s, peak.value) if w.cfg in ("c1", "c2") else
                        ozaki_roofline(w, i8_ms.value, i8_ops.value, i8_n.value, achieved, g_n.value,
                                       peak.value, args.moduli, i8_peak) if ozaki else
                        {"bound": "tensor", "achieved": achieved, "peak": peak.value,
                         "unit": "TFLOP/s", "frac": (achieved / peak.value) if achieved else None,
                         "traffic": ncu_traffic(w), "kernel": "gemm_f64_tma_kernel",
                         "launches": g_n.value,
                         "peak_source": "measured live before the timed region: DMMA m8n8k4 register-only probe (si_dmma_peak); MEASURED_PEAKS.json has no FP64 entry"},
            "fp64_dmma": fp64_dmma,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "gpu_launches": launches.value,
            "setup_s": getattr(w, "setup_s", None),
            "hbm_peak_gb": torch.cuda.max_memory_allocated() / 1e9,
            "clocks": clocks,
        }
        if COMM_FALLBACK:
            line["comm_fallback"] = ("peer exchange unavailable, NCCL all-gather used: "
                                     + COMM_FALLBACK["reason"])
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None,
                    help="timed steps (default: 5; our arm's c1 / c2 / c3 default to 15000 / "
                         "120 / 300 so the timed region is >= 2 s and the clock sampler sees it)")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=["c1", "c2", "c3", "c4", "c5"], default="c4")
    ap.add_argument("--n", "--size", dest="n", type=int, default=None)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--hoist", action="store_true",
                    help="c4 only, opt-in labelled variant: hoist the state-independent "
                         "composite parts (NOT the reference DAG; FLOPs counted as executed)")
    ap.add_argument("--comm", choices=["peer", "peer-stream", "nccl", "native"], default="peer",
                    help="row-panel exchange of the sharded path (N > 1); native = the "
                         "library's own block-row engine behind si_sharded_* (NCCL)")
    ap.add_argument("--shard", choices=["rows", "parts"], default="rows",
                    help="c4 at N > 1: block-row sharding of every product (rows) or the "
                         "composite parts on GPU groups + one tree reduction (parts)")
    ap.add_argument("--gemm", choices=["auto", "dmma", "ozaki"], default="auto",
                    help="FP64 product backend of the dense configs c3/c4/c5: FP64 DMMA, or "
                         "Ozaki-II emulation on the INT8 tensor cores (si_set_gemm_backend); "
                         "auto = ozaki")
    ap.add_argument("--moduli", type=int, default=16,
                    help="--gemm ozaki: number of moduli (16 = at least DGEMM's accuracy)")
    ap.add_argument("--i8-kernel", choices=["auto", "pair", "single", "multicast"], default="auto",
                    help="--gemm ozaki: INT8 tensor-core kernel (CTA pairs or single CTAs)")
    ap.add_argument("--no-dmma-side", action="store_true",
                    help="--gemm ozaki: skip the FP64 DMMA reference point timed after the run")
    ap.add_argument("--streams", action="store_true",
                    help="c4: evaluate the composite parts on concurrent CUDA streams (the "
                         "paper's simultaneously evaluated parts, on one GPU; bitwise equal)")
    ap.add_argument("--ref-budget", type=float, default=300.0,
                    help="--impl reference, c4/c5: wall-clock budget (s) for the executed "
                         "full-size CPU steps (at least one is always executed)")
    args = ap.parse_args()
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    if args.steps is None:
        short = {"c1": 15000, "c2": 120, "c3": 300}  # sub-20-ms steps: a >= 2 s timed region
        args.steps = short.get(args.config, 5) if args.impl == "ours" else 5
    if args.steps < 1:
        ap.error("--steps must be >= 1")
    env_world = os.environ.get("WORLD_SIZE")
    if env_world is None and args.gpus > 1:
        # not launched by torchrun: start the N ranks ourselves (one per GPU)
        return launch_ranks(args.gpus)
    if env_world is not None and int(env_world) != args.gpus:
        print(json.dumps({"error": f"--gpus {args.gpus} but WORLD_SIZE={env_world}: "
                                   "launch one rank per GPU with --nproc-per-node equal to --gpus"}),
              flush=True)
        return 2
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


def launch_ranks(n: int) -> int:
    """`bench.py --gpus N` without torchrun: re-launch this command under
    torch.distributed.run with N ranks on this node (127.0.0.1 rendezvous)."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)]
    cmd += sys.argv[1:]
    return subprocess.call(cmd)


if __name__ == "__main__":
    sys.exit(main())
