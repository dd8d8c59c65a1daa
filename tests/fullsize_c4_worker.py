"""Worker of tests/test_gpu_fullsize.py::test_c4_full_size_two_iterations_vs_oracle.

BASELINE config 4 at its full size (n=16384, 64 RHS): two iterations of plain
Richardson + composite_step((2,3,4,5), 2) on the GPU (the bench's kernels), the
same two on the GPU for the permutation-similar Pi A Pi^T (the noise floor),
the same two with the Ozaki-II INT8 backend (bench.py --gemm ozaki),
then the CPU oracle on the host cores (~2 min per iteration).  Started by
conftest.py as soon as collection finishes, so the host-bound oracle overlaps
the other GPU tests; the test waits for the JSON this writes to <out>/result.json.

    python tests/fullsize_c4_worker.py <out_dir>
"""

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402


def _rel_t(x, ref):
    d = torch.linalg.norm(ref).item()
    return torch.linalg.norm(x - ref).item() / (d if d > 0 else 1.0)


def _rel_np(x, ref):
    d = np.linalg.norm(ref)
    return float(np.linalg.norm(x - ref) / (d if d > 0 else 1.0))


def _gpu_c4(P, a, b, iters):
    sp = P.split_scalar(a, P.inf_norm(a) / 2.0, check_pd=False, verify=False)
    st = P.initial_series(sp, 0, 1, order=2)
    theta = torch.zeros_like(b)
    spec = P.CompositeSpec((2, 3, 4, 5))
    for _ in range(iters):
        theta = P.plain_richardson(theta, st.estimate, sp.matrix, b, st.ctr)
        st = P.composite_step(st, sp.matrix, sp, spec, 2)
        yield st.estimate, theta, st.ctr


def main():
    out = sys.argv[1]
    import paper_2008_11480_b200 as P
    from oracle import seriesinv_oracle as O
    from paper_2008_11480_b200 import _lib, configs

    n, rhs, iters = 16384, 64, 2
    res = {"n": n, "rhs": rhs, "iters": iters}
    a, b = configs.c4_householder_device(n=n, rhs=rhs)
    lam, _, _ = configs._c4_draws(n, 64, rhs, 0)
    res["kappa"] = float(lam.max() / lam.min())  # A = Q diag(lam) Q^T, Q orthogonal
    gpu = []
    for p, t, ctr in _gpu_c4(P, a, b, iters):
        gpu.append((p.cpu().numpy(), t.cpu().numpy()))
    res["gpu_ctr"] = [ctr.mmm, ctr.mvm]
    perm = np.random.default_rng(17).permutation(n)
    pt = torch.as_tensor(perm, device=a.device)
    floor = 0.0
    for k, (p, t, _) in enumerate(_gpu_c4(P, a[pt][:, pt].contiguous(), b[pt], iters)):
        pu = torch.empty_like(p)
        pu[pt[:, None], pt[None, :]] = p
        tu = torch.empty_like(t)
        tu[pt] = t
        pd = torch.as_tensor(gpu[k][0], device=a.device)
        td = torch.as_tensor(gpu[k][1], device=a.device)
        floor = max(floor, _rel_t(pu, pd), _rel_t(tu, td))
        del pu, tu, pd, td, p, t
    res["floor"] = floor
    # the same two iterations with every n x n product emulated on the INT8
    # tensor cores (Ozaki-II, 16 moduli: the bench's --gemm ozaki)
    oz = []
    with P.gemm_backend("ozaki", moduli=16, min_dim=1024):
        for p, t, ctr in _gpu_c4(P, a, b, iters):
            oz.append((p.cpu().numpy(), t.cpu().numpy()))
    res["ozaki_ctr"] = [ctr.mmm, ctr.mvm]
    res["ozaki_vs_dmma"] = [max(_rel_np(o[0], g[0]), _rel_np(o[1], g[1])) for o, g in zip(oz, gpu)]
    a_np, b_np = a.cpu().numpy(), b.cpu().numpy()
    del a, b, pt
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    _lib.call("si_trim", _lib.handle(0))  # the GPU is free for the other tests now
    osp = O.split_scalar(a_np, O.inf_norm(a_np) / 2.0)
    del a_np
    ost = O.initial_series(osp, 0, 1, 2)
    oth = np.zeros_like(b_np)
    res["per_iteration"] = []
    for k in range(iters):
        oth = O.plain_richardson(oth, ost.estimate, osp.matrix, b_np, ost.ctr)
        ost = O.composite_step(ost, osp.matrix, osp, (2, 3, 4, 5), 2)
        res["per_iteration"].append([_rel_np(gpu[k][0], ost.estimate), _rel_np(gpu[k][1], oth)])
        res.setdefault("per_iteration_ozaki", []).append(
            [_rel_np(oz[k][0], ost.estimate), _rel_np(oz[k][1], oth)])
    res["oracle_ctr"] = [ost.ctr.mmm, ost.ctr.mvm]
    with open(os.path.join(out, "result.json.tmp"), "w") as fh:
        json.dump(res, fh)
    os.replace(os.path.join(out, "result.json.tmp"), os.path.join(out, "result.json"))


if __name__ == "__main__":
    main()
