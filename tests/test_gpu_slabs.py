"""GPU parity of the multi-rank z-slab path on ONE device.

The ranks are threads of this process sharing cuda:0 through libfem's in-process
transport (fem_local_group_create): every collective is device-to-device copies
ordered by events between the ranks' streams, never a kernel waiting on another
(B200_PROFILING.md: emulate ranks without device-side waits).  The partitioned
operator, diagonal, load vector, transfers, V-cycle and PCG are compared with the
single-rank handle (itself pinned to the oracle by test_gpu_cg / test_gpu_sipg)
and, for the operator, with the CPU oracle directly.

Bars: operator / diagonal / transfers <= 1e-12 relative max-norm (only the
summation order of shared-node contributions differs), V-cycle <= 1e-11 with
lambda pinned, PCG iterations +-1 and the oracle-checked true residual.
"""
import threading

import numpy as np
import pytest
import torch

import fem_inputs
from oracle import cg as ocg, sipg as osipg
from oracle.mesh import Mesh, CG, SIPG, DIRICHLET, NEUMANN

pytestmark = pytest.mark.gpu

MIXED = (DIRICHLET, NEUMANN, DIRICHLET, DIRICHLET, NEUMANN, DIRICHLET)


def fem_mod():
    from paper_1611_03029_b200 import fem
    return fem


def relmax(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


def run_ranks(P, make_kw, body):
    """Run body(F, rank) on P threads, each with its own rank handle and stream."""
    fem = fem_mod()
    group = fem.LocalGroup(P)
    out, errs = [None] * P, []

    def worker(r):
        try:
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                F = fem.Fem(rank=r, nranks=P, local_group=group, stream=s, **make_kw)
                try:
                    out[r] = body(F, r)
                finally:
                    F.fem_sync()
                    F.close()
        except Exception as e:  # noqa: BLE001 - reported below
            errs.append((r, e))

    th = [threading.Thread(target=worker, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    group.close()
    assert not errs, errs
    return out


def own_slices(F1, P, make_kw, level=None):
    """(first, n_owned) of every rank for the finest level (or `level`)."""
    fem = fem_mod()
    parts = [fem.partition(make_kw["cells"], make_kw["degree"], make_kw.get("method", fem.FEM_CG), r, P,
                           slab_min_layers=make_kw.get("slab_min_layers"), slab_min_dofs=0) for r in range(P)]
    lv = -1 if level is None else level
    return [(p[lv]["first_global"], p[lv]["n_owned"]) for p in parts]


CASES = [
    # method, k, cells, eps, bc, P, slab_min_layers
    ("cg", 2, (2, 4, 6), 0.05, MIXED, 2, 1),
    ("cg", 3, (4, 4, 8), 0.0, (DIRICHLET,) * 6, 4, 1),
    ("cg", 4, (4, 2, 6), 0.05, (DIRICHLET,) * 6, 3, 2),
    ("sipg", 2, (2, 2, 6), 0.05, MIXED, 2, 1),
    ("sipg", 3, (4, 4, 8), 0.0, (DIRICHLET,) * 6, 4, 1),
    ("sipg", 4, (2, 2, 4), 0.05, (DIRICHLET,) * 6, 2, 2),
    # eight ranks (one z-layer each on the finest level, the box's GPU count)
    ("cg", 2, (2, 2, 8), 0.05, MIXED, 8, 1),
    ("sipg", 2, (2, 2, 8), 0.0, (DIRICHLET,) * 6, 8, 1),
]


def kw_of(method, k, cells, eps, bc, mnl):
    fem = fem_mod()
    return dict(cells=cells, degree=k, method=fem.FEM_CG if method == "cg" else fem.FEM_SIPG,
                deform_eps=eps, bc=bc, slab_min_layers=mnl, slab_min_dofs=0)


@pytest.mark.parametrize("method,k,cells,eps,bc,P,mnl", CASES)
def test_apply_diagonal_rhs_match_single_rank_and_oracle(method, k, cells, eps, bc, P, mnl):
    fem = fem_mod()
    kw = kw_of(method, k, cells, eps, bc, mnl)
    F1 = fem.Fem(**kw)
    n = F1.n_global
    x = fem_inputs.uniform_pm1(11, n)
    y1 = np.zeros(n)
    F1.fem_apply(x, y1)
    d1 = np.zeros(n)
    F1.fem_diagonal(d1)
    b1 = np.zeros(n)
    F1.fem_rhs(b1)
    F1.close()
    sl = own_slices(F1, P, kw)

    def body(F, r):
        f, m = sl[r]
        assert (F.first_global, F.n_local, F.n_global) == (f, m, n)
        xr = torch.from_numpy(x[f:f + m]).cuda()
        yr, dr, br = torch.zeros_like(xr), torch.zeros_like(xr), torch.zeros_like(xr)
        F.fem_apply(xr, yr)
        F.fem_diagonal(dr)
        F.fem_rhs(br)
        F.fem_sync()
        return yr.cpu().numpy(), dr.cpu().numpy(), br.cpu().numpy()

    res = run_ranks(P, kw, body)
    y, d, b = (np.concatenate([res[r][i] for r in range(P)]) for i in range(3))
    assert relmax(y, y1) <= 1e-12
    assert relmax(d, d1) <= 1e-12
    assert relmax(b, b1) <= 1e-12
    m = Mesh(cells, k, eps=eps, bc=bc)
    yo = ocg.apply(m, x) if method == "cg" else osipg.apply(m, x)
    assert relmax(y, yo) <= 1e-12


@pytest.mark.parametrize("method,k,cells,eps,bc,P,mnl", CASES)
def test_levels_and_transfers_match_single_rank(method, k, cells, eps, bc, P, mnl, monkeypatch):
    # the single-rank reference uses the element-form CG transfers, the ranks the node-grid form
    # (both forms against the oracle: test_gpu_cg.py)
    monkeypatch.setenv("FEM_GT_MIN_CELLS", "1000000000")
    fem = fem_mod()
    kw = kw_of(method, k, cells, eps, bc, mnl)
    F1 = fem.Fem(**kw)
    nl = F1.n_levels
    parts = [fem.partition(cells, k, kw["method"], r, P, slab_min_layers=mnl, slab_min_dofs=0) for r in range(P)]
    ref = {}
    for l in range(nl):
        ng = parts[0][l]["n_global"]
        x = fem_inputs.uniform_pm1(30 + l, ng)
        y = np.zeros(ng)
        F1.fem_level_apply(l, x, y)
        d = np.zeros(ng)
        F1.fem_level_diagonal(l, d)
        ref[("apply", l)], ref[("diag", l)] = y, d
        if l >= 1:
            ref[("lam", l)] = F1.fem_level_lambda(l)
            nc = parts[0][l - 1]["n_global"]
            xc = fem_inputs.uniform_pm1(50 + l, nc)
            xf = fem_inputs.uniform_pm1(70 + l, ng)
            pf = xf.copy()
            F1.mg_prolongate_add(l, xc, pf)
            rc = np.zeros(nc)
            F1.mg_restrict(l, xf, rc)
            ref[("prol", l)], ref[("rest", l)] = pf, rc
    F1.close()
    monkeypatch.setenv("FEM_GT_MIN_CELLS", "1")

    def body(F, r):
        got = {}
        for l in range(nl):
            q = parts[r][l]
            f, m, ng = q["first_global"], q["n_owned"], q["n_global"]
            x = fem_inputs.uniform_pm1(30 + l, ng)[f:f + m].copy()
            y = np.zeros(m)
            F.fem_level_apply(l, x, y)
            d = np.zeros(m)
            F.fem_level_diagonal(l, d)
            got[("apply", l)], got[("diag", l)] = y, d
            if l >= 1:
                got[("lam", l)] = F.fem_level_lambda(l)
                qc = parts[r][l - 1]
                xc = fem_inputs.uniform_pm1(50 + l, qc["n_global"])
                xc = xc[qc["first_global"]:qc["first_global"] + qc["n_owned"]].copy()
                pf = fem_inputs.uniform_pm1(70 + l, ng)[f:f + m].copy()
                F.mg_prolongate_add(l, xc, pf)
                xf = fem_inputs.uniform_pm1(70 + l, ng)[f:f + m].copy()
                rc = np.zeros(qc["n_owned"])
                F.mg_restrict(l, xf, rc)
                got[("prol", l)], got[("rest", l)] = pf, rc
        return got

    res = run_ranks(P, kw, body)
    for l in range(nl):
        for key in ("apply", "diag", "prol", "rest"):
            if (key, l) not in ref:
                continue
            lev = l - 1 if key == "rest" else l
            if parts[0][lev]["distributed"]:
                got = np.concatenate([res[r][(key, l)] for r in range(P)])
            else:       # replicated level: every rank holds the whole vector
                got = res[0][(key, l)]
                for r in range(1, P):
                    assert relmax(res[r][(key, l)], got) <= 1e-12
            assert relmax(got, ref[(key, l)]) <= 1e-12, (key, l)
        if l >= 1:
            for r in range(P):
                assert abs(res[r][("lam", l)] - ref[("lam", l)]) <= 1e-10 * ref[("lam", l)]


@pytest.mark.parametrize("method,k,cells,eps,bc,P,mnl", CASES)
def test_vcycle_and_pcg_match_single_rank(method, k, cells, eps, bc, P, mnl):
    fem = fem_mod()
    kw = kw_of(method, k, cells, eps, bc, mnl)
    F0 = fem.Fem(**kw)
    lam = [0.0] + [F0.fem_level_lambda(l) for l in range(1, F0.n_levels)]
    n = F0.n_global
    F0.close()
    kw_l = dict(kw, lambda_override=lam)
    F1 = fem.Fem(**kw_l)
    r0 = fem_inputs.uniform_pm1(5, n)
    z1 = np.zeros(n)
    F1.mg_vcycle(r0, z1)
    b = np.zeros(n)
    F1.fem_rhs(b)
    x1 = np.zeros(n)
    its1, rr1, ok1 = F1.cg_solve(b, x1, rtol=1e-10)
    assert ok1
    F1.close()
    sl = own_slices(F1, P, kw)

    def body(F, r):
        f, m = sl[r]
        z = np.zeros(m)
        F.mg_vcycle(r0[f:f + m].copy(), z)
        bb = torch.zeros(m, dtype=torch.float64, device="cuda")
        F.fem_rhs(bb)
        xx = torch.zeros_like(bb)
        its, rr, ok = F.cg_solve(bb, xx, rtol=1e-10)
        return z, xx.cpu().numpy(), its, rr, ok

    res = run_ranks(P, kw_l, body)
    z = np.concatenate([res[r][0] for r in range(P)])
    assert relmax(z, z1) <= 1e-11
    its = {res[r][2] for r in range(P)}
    assert len(its) == 1, "ranks disagree on the iteration count"
    assert abs(its.pop() - its1) <= 1
    assert all(res[r][4] and res[r][3] <= 1e-10 for r in range(P))
    x = np.concatenate([res[r][1] for r in range(P)])
    m_ = Mesh(cells, k, eps=eps, bc=bc)
    ax = ocg.apply(m_, x) if method == "cg" else osipg.apply(m_, x)
    bb = b
    assert np.linalg.norm(bb - ax) / np.linalg.norm(bb) <= 1e-9


@pytest.mark.parametrize("method,k,cells,P", [("cg", 3, (2, 4, 6), 2), ("sipg", 2, (4, 2, 4), 2)])
def test_shell_variable_kappa_slabs_match_single_rank_and_oracle(method, k, cells, P):
    """N3 on z-slabs: the shell patch coordinates use the GLOBAL z cell index and count."""
    fem = fem_mod()
    kw = kw_of(method, k, cells, 0.0, (DIRICHLET,) * 6, 1)
    kw.update(geometry=fem.FEM_GEOM_SHELL, mapping_degree=5, kappa_amplitude=0.5)
    F1 = fem.Fem(**kw)
    n = F1.n_global
    x = fem_inputs.uniform_pm1(13, n)
    y1, d1, b1 = np.zeros(n), np.zeros(n), np.zeros(n)
    F1.fem_apply(x, y1)
    F1.fem_diagonal(d1)
    F1.fem_rhs(b1)
    its1, _, ok1 = F1.cg_solve(b1, np.zeros(n))
    F1.close()
    sl = own_slices(F1, P, kw)

    def body(F, r):
        f, m = sl[r]
        xr = torch.from_numpy(x[f:f + m]).cuda()
        yr, dr, br = torch.zeros_like(xr), torch.zeros_like(xr), torch.zeros_like(xr)
        F.fem_apply(xr, yr)
        F.fem_diagonal(dr)
        F.fem_rhs(br)
        its, _, ok = F.cg_solve(br, torch.zeros_like(xr))
        F.fem_sync()
        return yr.cpu().numpy(), dr.cpu().numpy(), br.cpu().numpy(), its, ok

    res = run_ranks(P, kw, body)
    y, d, b = (np.concatenate([res[r][i] for r in range(P)]) for i in range(3))
    assert relmax(y, y1) <= 1e-12 and relmax(d, d1) <= 1e-12 and relmax(b, b1) <= 1e-12
    m = Mesh(cells, k, geometry=1, mapping_degree=5, kappa_amp=0.5)
    assert relmax(y, ocg.apply(m, x) if method == "cg" else osipg.apply(m, x)) <= 1e-12
    assert ok1 and all(res[r][4] for r in range(P))
    assert all(abs(res[r][3] - its1) <= 1 for r in range(P))
