"""Multi-rank z-slab host logic on CPU: gloo, world_size 2 and 3.

No GPU is involved.  Each process is one rank; it asks libfem's host-only
fem_partition for its slab of every level, and

1. the ranks' descriptions are checked against each other (owned ranges tile the
   global vector in rank order, the ghost of a rank is the first owned plane /
   adjacent layer of its neighbour, replicated levels hold everything, distributed
   levels form a prefix of the hierarchy);
2. the exchange protocol of include/fem.h is run with gloo point-to-point on the
   oracle's element-wise operator restricted to the rank's cells: CG imports the
   ghost node plane from the rank above, applies its cells into owned + ghost
   storage and compress-adds the ghost plane into the owner; SIPG imports one ghost
   cell layer from each neighbour.  The gathered owned slices must equal the
   global oracle apply, and the gathered transfer-level residual (all-reduce of
   zero-padded owned slices) must equal the global vector.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(rank, world, port, case, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        _check_rank(rank, world, case)
        q.put((rank, None))
    except Exception as e:  # noqa: BLE001 - sent to the parent
        import traceback
        q.put((rank, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


def _exchange(sends, recvs):
    """sends/recvs: lists of (peer, tensor); one message per direction per pair."""
    reqs = [dist.isend(t, peer) for peer, t in sends] + [dist.irecv(t, peer) for peer, t in recvs]
    for r in reqs:
        r.wait()


def _check_rank(rank, P, case):
    import fem_inputs
    from oracle import cg as ocg, sipg as osipg
    from oracle.mesh import Mesh
    from paper_1611_03029_b200 import fem

    method, k, cells, eps, mnl = case
    meth = fem.FEM_CG if method == "cg" else fem.FEM_SIPG
    parts = fem.partition(cells, k, meth, rank, P, slab_min_layers=mnl, slab_min_dofs=0)
    allp = [None] * P
    dist.all_gather_object(allp, parts)

    # ---- 1. partition consistency
    nl = len(parts)
    seen_replicated = False
    for l in range(nl - 1, -1, -1):          # finest first
        lv = [allp[r][l] for r in range(P)]
        if lv[0]["distributed"]:
            assert not seen_replicated, "distributed levels must be a prefix of the hierarchy"
            off = 0
            for r in range(P):
                assert lv[r]["first_global"] == off
                off += lv[r]["n_owned"]
                assert lv[r]["ghost_lo"] == (r - 1 if r > 0 else -1)
                assert lv[r]["ghost_hi"] == (r + 1 if r < P - 1 else -1)
                assert lv[r]["cell_z0"] == r * lv[r]["cells"][2]
                assert lv[r]["cells"][2] * P == lv[r]["global_cells"][2]
                assert lv[r]["cells"][2] >= (1 if l == nl - 1 else mnl)
            assert off == lv[0]["n_global"]
        else:
            seen_replicated = True
            for r in range(P):
                assert lv[r]["n_owned"] == lv[r]["n_stored"] == lv[r]["n_global"]
                assert lv[r]["first_global"] == 0 and lv[r]["ghost_lo"] == lv[r]["ghost_hi"] == -1
    assert allp[0][nl - 1]["distributed"] and not allp[0][0]["distributed"]

    # ---- 2. exchange protocol on the oracle operator, finest level
    q = parts[-1]
    m = Mesh(cells, k, eps=eps)
    n, f, no, ns = q["n_global"], q["first_global"], q["n_owned"], q["n_stored"]
    x = fem_inputs.uniform_pm1(21, n)
    nzl, z0 = q["cells"][2], q["cell_z0"]
    my_cells = np.arange(z0 * cells[0] * cells[1], (z0 + nzl) * cells[0] * cells[1])
    if method == "cg":
        plane = (k * cells[0] + 1) * (k * cells[1] + 1)
        assert ns - no == (plane if rank < P - 1 else 0)
        xs = torch.zeros(ns, dtype=torch.float64)
        xs[:no] = torch.from_numpy(x[f:f + no])
        snd = [(rank - 1, xs[:plane].clone())] if rank > 0 else []
        rcv = [(rank + 1, torch.zeros(plane, dtype=torch.float64))] if rank < P - 1 else []
        _exchange(snd, rcv)
        if rcv:
            xs[no:] = rcv[0][1]
        xsn = xs.numpy()
        assert np.array_equal(xsn, x[f:f + ns]), "ghost plane = the neighbour's first owned plane"
        mask = m.cg_dirichlet_mask()
        op = ocg.Operator(m)
        dm = m.cg_dofmap(my_cells) - f          # local storage indices
        assert dm.min() >= 0 and dm.max() < ns
        xe = np.where(mask[dm + f], 0.0, xsn[dm])
        G = np.broadcast_to(op.G0, (len(my_cells),) + op.G0.shape[1:]) if op.uniform \
            else ocg.metric(m, my_cells, op.quad)
        ye = ocg.element_apply_G(G, xe, op.quad)
        ys = torch.from_numpy(np.bincount(dm.ravel(), weights=ye.ravel(), minlength=ns))
        snd = [(rank + 1, ys[no:].clone())] if rank < P - 1 else []
        rcv = [(rank - 1, torch.zeros(plane, dtype=torch.float64))] if rank > 0 else []
        _exchange(snd, rcv)
        if rcv:
            ys[:plane] += rcv[0][1]
        y_own = np.where(mask[f:f + no], x[f:f + no], ys[:no].numpy())
        y_ref = ocg.apply(m, x)
    else:
        N3 = (k + 1) ** 3
        layer = cells[0] * cells[1] * N3
        assert ns - no == 2 * layer and no == nzl * layer
        lo = torch.zeros(layer, dtype=torch.float64)
        hi = torch.zeros(layer, dtype=torch.float64)
        own = torch.from_numpy(x[f:f + no].copy())
        snd, rcv = [], []
        if rank > 0:
            snd.append((rank - 1, own[:layer].clone()))
            rcv.append((rank - 1, lo))
        if rank < P - 1:
            snd.append((rank + 1, own[no - layer:].clone()))
            rcv.append((rank + 1, hi))
        _exchange(snd, rcv)
        xg = np.zeros(n)                         # what the rank can see: own + ghost layers
        xg[f:f + no] = own.numpy()
        if rank > 0:
            xg[f - layer:f] = lo.numpy()
            assert np.array_equal(lo.numpy(), x[f - layer:f])
        if rank < P - 1:
            xg[f + no:f + no + layer] = hi.numpy()
            assert np.array_equal(hi.numpy(), x[f + no:f + no + layer])
        y_own = osipg.apply_cells(m, xg, my_cells).ravel()
        y_ref = osipg.apply(m, x)
    got = [None] * P
    dist.all_gather_object(got, y_own)
    y = np.concatenate(got)
    assert np.abs(y - y_ref).max() <= 1e-12 * np.abs(y_ref).max()

    # ---- 3. gather of the last distributed level (all-reduce of zero-padded owned slices)
    for l in range(nl - 1, 0, -1):
        if allp[0][l]["distributed"] and not allp[0][l - 1]["distributed"]:
            ql = parts[l]
            v = fem_inputs.uniform_pm1(40 + l, ql["n_global"])
            full = torch.zeros(ql["n_global"], dtype=torch.float64)
            a, b = ql["first_global"], ql["first_global"] + ql["n_owned"]
            full[a:b] = torch.from_numpy(v[a:b])
            dist.all_reduce(full)
            assert np.array_equal(full.numpy(), v)


CASES = [
    ("cg", 2, (2, 2, 6), 0.05, 1),
    ("cg", 3, (2, 2, 8), 0.0, 2),
    ("sipg", 2, (2, 4, 6), 0.05, 1),
    ("sipg", 3, (2, 2, 4), 0.0, 1),
]


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("case", CASES)
def test_slab_partition_and_exchange_gloo(world, case):
    if case[2][2] % world:
        pytest.skip("n_z not divisible by world size")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_run, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    errs = [e for _, e in res if e]
    assert not errs, "\n".join(errs)


def test_partition_rejects_indivisible_slabs():
    import sys
    sys.path.insert(0, ROOT)
    from paper_1611_03029_b200 import fem
    with pytest.raises(fem.FemError):
        fem.partition((4, 4, 6), 2, fem.FEM_CG, 0, 4)
    p1 = fem.partition((4, 4, 8), 2, fem.FEM_CG, 0, 1)
    assert all(not q["distributed"] and q["n_owned"] == q["n_global"] for q in p1)
