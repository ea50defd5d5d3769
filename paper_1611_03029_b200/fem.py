"""Thin ctypes binding of libfem (include/fem.h): argument marshalling only.

Every step of the hot path runs in libfem's CUDA kernels; this module converts
torch tensors / numpy arrays to (pointer, length) pairs and return codes to
exceptions.  There is no fallback: if libfem.so is missing or fails to load,
importing the binding raises.

Names follow the C ABI: fem_setup -> Fem(...), fem_apply -> Fem.fem_apply, etc.
Vectors may be CUDA tensors (used in place, asynchronous on the handle's
stream) or host numpy arrays / CPU tensors (staged by libfem, synchronous).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FEM_LIB", os.path.join(_HERE, "libfem.so"))   # FEM_LIB: experiment builds

FEM_OK, FEM_NOT_CONVERGED = 0, 1
ERRORS = {-1: "FEM_E_ARG", -2: "FEM_E_SIZE", -3: "FEM_E_GEOMETRY", -4: "FEM_E_BREAKDOWN",
          -5: "FEM_E_CUDA", -6: "FEM_E_NCCL", -7: "FEM_E_OOM"}
FEM_CG, FEM_SIPG = 0, 1
FEM_BC_DIRICHLET, FEM_BC_NEUMANN = 0, 1
FEM_GEOM_BOX, FEM_GEOM_SHELL = 0, 1


class FemError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{ERRORS.get(code, code)}: {msg}")
        self.code = code


class fem_mesh(C.Structure):
    _fields_ = [("n", C.c_int32 * 3), ("lo", C.c_double * 3), ("hi", C.c_double * 3),
                ("deform_eps", C.c_double), ("bc", C.c_int32 * 6), ("rank", C.c_int32),
                ("nranks", C.c_int32), ("nccl_id", C.c_void_p), ("local_group", C.c_void_p),
                ("geometry", C.c_int32), ("mapping_degree", C.c_int32), ("kappa_amplitude", C.c_double)]


class fem_options(C.Structure):
    _fields_ = [("penalty_factor", C.c_double), ("cheb_degree", C.c_int32),
                ("cheb_lo", C.c_double), ("cheb_hi", C.c_double), ("eig_iters", C.c_int32),
                ("coarse_cells", C.c_int32), ("eig_seed", C.c_uint64),
                ("lambda_override", C.POINTER(C.c_double)), ("stream", C.c_void_p),
                ("device", C.c_int32), ("profile", C.c_int32), ("slab_min_layers", C.c_int32),
                ("slab_min_dofs", C.c_int64)]


class fem_level_part(C.Structure):
    _fields_ = [("cells", C.c_int32 * 3), ("global_cells", C.c_int32 * 3), ("cell_z0", C.c_int32),
                ("distributed", C.c_int32), ("n_owned", C.c_int64), ("first_global", C.c_int64),
                ("n_global", C.c_int64), ("n_stored", C.c_int64), ("ghost_lo", C.c_int32),
                ("ghost_hi", C.c_int32)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libfem.so not built ({LIB_PATH}); run `python -m paper_1611_03029_b200.build`")
    lib = C.CDLL(LIB_PATH)
    P, I32, I64, D = C.c_void_p, C.c_int32, C.c_int64, C.c_double
    sig = {
        "fem_default_options": (C.c_int, [C.POINTER(fem_options)]),
        "fem_setup": (C.c_int, [C.POINTER(fem_mesh), I32, I32, C.POINTER(fem_options), C.POINTER(P)]),
        "fem_partition": (C.c_int, [C.POINTER(fem_mesh), I32, I32, C.POINTER(fem_options),
                                    C.POINTER(fem_level_part), I32, C.POINTER(I32)]),
        "fem_nccl_unique_id": (C.c_int, [P, I64]),
        "fem_local_group_create": (C.c_int, [I32, C.POINTER(P)]),
        "fem_local_group_destroy": (None, [P]),
        "fem_info": (C.c_int, [P, C.POINTER(I64), C.POINTER(I64), C.POINTER(I64), C.POINTER(I32)]),
        "fem_apply": (C.c_int, [P, P, I64, P, I64]),
        "fem_diagonal": (C.c_int, [P, P, I64]),
        "mg_vcycle": (C.c_int, [P, P, I64, P, I64]),
        "cg_solve": (C.c_int, [P, P, I64, P, I64, D, I32, C.POINTER(I32), C.POINTER(D)]),
        "cg_solve_zero": (C.c_int, [P, P, I64, P, I64, D, I32, C.POINTER(I32), C.POINTER(D)]),
        "fem_rhs": (C.c_int, [P, P, I64]),
        "cg_history": (C.c_int, [P, C.POINTER(D), I32, C.POINTER(I32)]),
        "fem_level_info": (C.c_int, [P, I32, C.POINTER(I64), C.POINTER(I32)]),
        "fem_level_apply": (C.c_int, [P, I32, P, I64, P, I64]),
        "fem_level_diagonal": (C.c_int, [P, I32, P, I64]),
        "fem_level_lambda": (C.c_int, [P, I32, C.POINTER(D)]),
        "fem_level_geometry": (C.c_int, [P, I32, P, I64]),
        "mg_smooth": (C.c_int, [P, I32, P, I64, P, I64, I32]),
        "mg_prolongate_add": (C.c_int, [P, I32, P, I64, P, I64]),
        "mg_restrict": (C.c_int, [P, I32, P, I64, P, I64]),
        "mg_coarse_solve": (C.c_int, [P, P, I64, P, I64]),
        "fem_sync": (C.c_int, [P]),
        "fem_kernel_launches": (I64, []),
        "fem_profile_read": (C.c_int, [P, C.POINTER(D), C.POINTER(I64), I32]),
        "fem_profile_read_bytes": (C.c_int, [P, C.POINTER(D), C.POINTER(I64), C.POINTER(D), I32]),
        "fem_profile_mode": (C.c_int, [P, I32]),
        "fem_last_error": (C.c_char_p, []),
        "fem_destroy": (None, [P]),
        # include/fem_hdg.h
        "hdg_setup": (C.c_int, [C.POINTER(fem_mesh), I32, D, P, C.POINTER(P)]),
        "hdg_info": (C.c_int, [P, C.POINTER(I64), C.POINTER(I64)]),
        "hdg_apply": (C.c_int, [P, P, I64, P, I64]),
        "hdg_diagonal": (C.c_int, [P, P, I64]),
        "hdg_rhs": (C.c_int, [P, P, I64]),
        "hdg_local_solve": (C.c_int, [P, P, I64, I32, P, I64, P, I64]),
        "hdg_mixed_apply": (C.c_int, [P, P, I64, P, I64]),
        "hdg_postprocess": (C.c_int, [P, P, I64, P, I64, P, I64]),
        "hdg_cg_solve": (C.c_int, [P, P, I64, P, I64, D, I32, C.POINTER(I32), C.POINTER(D)]),
        "hdg_destroy": (None, [P]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype, f.argtypes = res, args
    return lib


_lib = _load()

# exported symbol list (tests check it against include/fem.h)
SYMBOLS = ("fem_default_options", "fem_setup", "fem_partition", "fem_nccl_unique_id",
           "fem_local_group_create", "fem_local_group_destroy", "fem_info", "fem_apply", "fem_diagonal", "mg_vcycle",
           "cg_solve", "cg_solve_zero", "cg_history", "fem_rhs", "fem_level_info", "fem_level_apply", "fem_level_diagonal",
           "fem_level_lambda", "fem_level_geometry", "mg_smooth", "mg_prolongate_add", "mg_restrict",
           "mg_coarse_solve", "fem_sync", "fem_kernel_launches", "fem_profile_read", "fem_profile_read_bytes", "fem_profile_mode",
           "fem_last_error",
           "fem_destroy", "hdg_setup", "hdg_info", "hdg_apply", "hdg_diagonal", "hdg_rhs", "hdg_local_solve",
           "hdg_mixed_apply", "hdg_postprocess", "hdg_cg_solve", "hdg_destroy")


def lib():
    return _lib


def kernel_launches() -> int:
    return int(_lib.fem_kernel_launches())


def _check(rc: int, allow=(FEM_OK,)):
    if rc not in allow:
        raise FemError(rc, _lib.fem_last_error().decode())
    return rc


def _vec(v, writable=False):
    """(pointer, length) of a contiguous float64 torch tensor or numpy array."""
    if hasattr(v, "data_ptr"):            # torch tensor
        import torch
        if v.dtype != torch.float64 or not v.is_contiguous():
            raise TypeError("vectors must be contiguous float64 tensors")
        return C.c_void_p(v.data_ptr()), v.numel()
    a = v
    if not isinstance(a, np.ndarray) or a.dtype != np.float64 or not a.flags["C_CONTIGUOUS"]:
        raise TypeError("vectors must be contiguous float64 numpy arrays or torch tensors")
    if writable and not a.flags["WRITEABLE"]:
        raise TypeError("output array is read-only")
    return C.c_void_p(a.ctypes.data), a.size


def nccl_unique_id() -> bytes:
    """fem_nccl_unique_id: 128 bytes to broadcast from one rank to all."""
    buf = C.create_string_buffer(128)
    _check(_lib.fem_nccl_unique_id(C.cast(buf, C.c_void_p), 128))
    return buf.raw


class LocalGroup:
    """fem_local_group_create: nranks threads of this process sharing one device."""

    def __init__(self, nranks: int):
        g = C.c_void_p()
        _check(_lib.fem_local_group_create(nranks, C.byref(g)))
        self.g, self.nranks = g, nranks

    def close(self):
        if getattr(self, "g", None):
            _lib.fem_local_group_destroy(self.g)
            self.g = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _mesh(cells, lo, hi, deform_eps, bc, rank, nranks, nccl_id, local_group, geometry=FEM_GEOM_BOX,
          mapping_degree=0, kappa_amplitude=0.0):
    m = fem_mesh()
    m.geometry, m.mapping_degree, m.kappa_amplitude = geometry, mapping_degree, kappa_amplitude
    m.n[:] = list(cells)
    m.lo[:] = list(lo)
    m.hi[:] = list(hi)
    m.deform_eps = deform_eps
    m.bc[:] = list(bc)
    m.rank, m.nranks = rank, nranks
    m.nccl_id = None
    m.local_group = local_group.g if local_group is not None else None
    return m


def _options(**kw):
    o = fem_options()
    _check(_lib.fem_default_options(C.byref(o)))
    for name, val in kw.items():
        if val is not None:
            setattr(o, name, val)
    return o


def partition(cells, degree, method=FEM_CG, rank=0, nranks=1, coarse_cells=None, slab_min_layers=None,
              slab_min_dofs=None):
    """fem_partition (host only): per level (coarsest first) a dict of the rank's slab."""
    m = _mesh(cells, (0.0,) * 3, (1.0,) * 3, 0.0, (FEM_BC_DIRICHLET,) * 6, rank, nranks, None, None)
    o = _options(coarse_cells=coarse_cells, slab_min_layers=slab_min_layers, slab_min_dofs=slab_min_dofs)
    out = (fem_level_part * 32)()
    nl = C.c_int32()
    _check(_lib.fem_partition(C.byref(m), degree, method, C.byref(o), out, 32, C.byref(nl)))
    res = []
    for i in range(nl.value):
        q = out[i]
        res.append({"cells": tuple(q.cells), "global_cells": tuple(q.global_cells), "cell_z0": q.cell_z0,
                    "distributed": bool(q.distributed), "n_owned": q.n_owned, "first_global": q.first_global,
                    "n_global": q.n_global, "n_stored": q.n_stored, "ghost_lo": q.ghost_lo,
                    "ghost_hi": q.ghost_hi})
    return res


class Fem:
    """One libfem handle (fem_setup ... fem_destroy).

    Multi-rank: pass rank/nranks and either nccl_id (bytes from nccl_unique_id(),
    one process per GPU) or local_group (LocalGroup shared by nranks threads)."""

    def __init__(self, cells, degree, method=FEM_CG, lo=(0.0, 0.0, 0.0), hi=(1.0, 1.0, 1.0),
                 deform_eps=0.0, bc=(FEM_BC_DIRICHLET,) * 6, penalty_factor=None, cheb_degree=None,
                 cheb_lo=None, cheb_hi=None, eig_iters=None, coarse_cells=None, eig_seed=None,
                 lambda_override=None, stream=None, device=None, profile=False, rank=0, nranks=1,
                 nccl_id=None, local_group=None, slab_min_layers=None, slab_min_dofs=None,
                 geometry=FEM_GEOM_BOX, mapping_degree=0, kappa_amplitude=0.0):
        m = _mesh(cells, lo, hi, deform_eps, bc, rank, nranks, None, local_group, geometry, mapping_degree,
                  kappa_amplitude)
        self._nccl_id = None
        if nccl_id is not None:
            self._nccl_id = C.create_string_buffer(bytes(nccl_id), 128)
            m.nccl_id = C.cast(self._nccl_id, C.c_void_p)
        self._group = local_group     # keep alive while the handle exists
        o = _options(penalty_factor=penalty_factor, cheb_degree=cheb_degree, cheb_lo=cheb_lo,
                     cheb_hi=cheb_hi, eig_iters=eig_iters, coarse_cells=coarse_cells, eig_seed=eig_seed,
                     slab_min_layers=slab_min_layers, slab_min_dofs=slab_min_dofs)
        self._lam = None
        if lambda_override is not None:
            self._lam = (C.c_double * len(lambda_override))(*lambda_override)
            o.lambda_override = C.cast(self._lam, C.POINTER(C.c_double))
        if stream is not None:
            o.stream = C.c_void_p(stream if isinstance(stream, int) else stream.cuda_stream)
        if device is not None:
            o.device = device
        o.profile = int(profile) if profile else 0   # True / 1: PCG applies, 2: finest smoother steps
        h = C.c_void_p()
        _check(_lib.fem_setup(C.byref(m), degree, method, C.byref(o), C.byref(h)))
        self.h = h
        self.degree, self.method, self.cells = degree, method, tuple(cells)
        nl, ng, fg, lv = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int32()
        _check(_lib.fem_info(h, C.byref(nl), C.byref(ng), C.byref(fg), C.byref(lv)))
        self.n_local, self.n_global, self.first_global, self.n_levels = nl.value, ng.value, fg.value, lv.value
        self.rank, self.nranks = rank, nranks

    def close(self):
        if getattr(self, "h", None):
            _lib.fem_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # ---- finest level
    def fem_apply(self, x, y):
        px, nx = _vec(x)
        py, ny = _vec(y, True)
        _check(_lib.fem_apply(self.h, px, nx, py, ny))
        return y

    def fem_diagonal(self, d):
        p, n = _vec(d, True)
        _check(_lib.fem_diagonal(self.h, p, n))
        return d

    def mg_vcycle(self, r, z):
        pr, nr = _vec(r)
        pz, nz = _vec(z, True)
        _check(_lib.mg_vcycle(self.h, pr, nr, pz, nz))
        return z

    def cg_solve(self, b, x, rtol=1e-10, maxit=1000):
        pb, nb = _vec(b)
        px, nx = _vec(x, True)
        its, rel = C.c_int32(), C.c_double()
        rc = _check(_lib.cg_solve(self.h, pb, nb, px, nx, rtol, maxit, C.byref(its), C.byref(rel)),
                    (FEM_OK, FEM_NOT_CONVERGED))
        return its.value, rel.value, rc == FEM_OK

    def cg_solve_zero(self, b, x, rtol=1e-10, maxit=1000):
        """cg_solve from x = 0; x is output only (a host x is not uploaded)."""
        pb, nb = _vec(b)
        px, nx = _vec(x, True)
        its, rel = C.c_int32(), C.c_double()
        rc = _check(_lib.cg_solve_zero(self.h, pb, nb, px, nx, rtol, maxit, C.byref(its), C.byref(rel)),
                    (FEM_OK, FEM_NOT_CONVERGED))
        return its.value, rel.value, rc == FEM_OK

    def cg_history(self):
        """||r_i|| / ||b||, i = 0 .. iterations, of the last cg_solve (host list)."""
        n = C.c_int32()
        _check(_lib.cg_history(self.h, None, 0, C.byref(n)))
        buf = (C.c_double * max(n.value, 1))()
        _check(_lib.cg_history(self.h, buf, n.value, C.byref(n)))
        return list(buf[:n.value])

    def fem_rhs(self, b):
        p, n = _vec(b, True)
        _check(_lib.fem_rhs(self.h, p, n))
        return b

    # ---- level-wise
    def level_info(self, level):
        n = C.c_int64()
        cells = (C.c_int32 * 3)()
        _check(_lib.fem_level_info(self.h, level, C.byref(n), cells))
        return n.value, tuple(cells)

    def fem_level_apply(self, level, x, y):
        px, nx = _vec(x)
        py, ny = _vec(y, True)
        _check(_lib.fem_level_apply(self.h, level, px, nx, py, ny))
        return y

    def fem_level_diagonal(self, level, d):
        p, n = _vec(d, True)
        _check(_lib.fem_level_diagonal(self.h, level, p, n))
        return d

    def fem_level_lambda(self, level):
        v = C.c_double()
        _check(_lib.fem_level_lambda(self.h, level, C.byref(v)))
        return v.value

    def fem_level_geometry(self, level, G):
        p, n = _vec(G, True)
        _check(_lib.fem_level_geometry(self.h, level, p, n))
        return G

    def mg_smooth(self, level, b, x, x_is_zero):
        pb, nb = _vec(b)
        px, nx = _vec(x, True)
        _check(_lib.mg_smooth(self.h, level, pb, nb, px, nx, 1 if x_is_zero else 0))
        return x

    def mg_prolongate_add(self, level, xc, xf):
        pc, nc = _vec(xc)
        pf, nf = _vec(xf, True)
        _check(_lib.mg_prolongate_add(self.h, level, pc, nc, pf, nf))
        return xf

    def mg_restrict(self, level, xf, xc):
        pf, nf = _vec(xf)
        pc, nc = _vec(xc, True)
        _check(_lib.mg_restrict(self.h, level, pf, nf, pc, nc))
        return xc

    def mg_coarse_solve(self, b, x):
        pb, nb = _vec(b)
        px, nx = _vec(x, True)
        _check(_lib.mg_coarse_solve(self.h, pb, nb, px, nx))
        return x

    def fem_sync(self):
        _check(_lib.fem_sync(self.h))

    def fem_profile_read(self, reset=False):
        ms, n = C.c_double(), C.c_int64()
        _check(_lib.fem_profile_read(self.h, C.byref(ms), C.byref(n), 1 if reset else 0))
        return ms.value, n.value

    def fem_profile_read_bytes(self, reset=False):
        ms, n, b = C.c_double(), C.c_int64(), C.c_double()
        _check(_lib.fem_profile_read_bytes(self.h, C.byref(ms), C.byref(n), C.byref(b), 1 if reset else 0))
        return ms.value, n.value, b.value

    def fem_profile_mode(self, mode):
        _check(_lib.fem_profile_mode(self.h, int(mode)))


class Hdg:
    """One HDG handle (include/fem_hdg.h: hdg_setup ... hdg_destroy), box meshes: Cartesian (fast
    diagonalization of the local inverse) or the deformed map (deform_eps != 0; the local inverse
    stored per cell, k <= 4).  Vectors are CUDA float64 tensors (device pointers only)."""

    def __init__(self, cells, degree, lo=(0.0, 0.0, 0.0), hi=(1.0, 1.0, 1.0), bc=(FEM_BC_DIRICHLET,) * 6,
                 tau=5.0, stream=None, deform_eps=0.0):
        m = _mesh(cells, lo, hi, deform_eps, bc, 0, 1, None, None)
        s = None if stream is None else C.c_void_p(stream if isinstance(stream, int) else stream.cuda_stream)
        h = C.c_void_p()
        _check(_lib.hdg_setup(C.byref(m), degree, tau, s, C.byref(h)))
        self.h = h
        self.degree, self.cells = degree, tuple(cells)
        nt, nc = C.c_int64(), C.c_int64()
        _check(_lib.hdg_info(h, C.byref(nt), C.byref(nc)))
        self.n_trace, self.n_cells = nt.value, nc.value
        self.n_cell_dofs = self.n_cells * (degree + 1) ** 3

    def close(self):
        if getattr(self, "h", None):
            _lib.hdg_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def hdg_apply(self, lam, y):
        pl, nl = _vec(lam)
        py, ny = _vec(y, True)
        _check(_lib.hdg_apply(self.h, pl, nl, py, ny))
        return y

    def hdg_diagonal(self, d):
        p, n = _vec(d, True)
        _check(_lib.hdg_diagonal(self.h, p, n))
        return d

    def hdg_rhs(self, r):
        p, n = _vec(r, True)
        _check(_lib.hdg_rhs(self.h, p, n))
        return r

    def hdg_local_solve(self, lam, u, q=None, with_f=True):
        pl, nl = _vec(lam)
        pu, nu = _vec(u, True)
        pq, nq = _vec(q, True) if q is not None else (None, 0)
        _check(_lib.hdg_local_solve(self.h, pl, nl, 1 if with_f else 0, pu, nu, pq, nq))
        return u

    def hdg_mixed_apply(self, qu, y):
        px, nx = _vec(qu)
        py, ny = _vec(y, True)
        _check(_lib.hdg_mixed_apply(self.h, px, nx, py, ny))
        return y

    def hdg_postprocess(self, q, u, ustar):
        pq, nq = _vec(q)
        pu, nu = _vec(u)
        ps, ns = _vec(ustar, True)
        _check(_lib.hdg_postprocess(self.h, pq, nq, pu, nu, ps, ns))
        return ustar

    def hdg_cg_solve(self, b, lam, rtol=1e-10, maxit=10000):
        pb, nb = _vec(b)
        px, nx = _vec(lam, True)
        its, rel = C.c_int32(), C.c_double()
        rc = _check(_lib.hdg_cg_solve(self.h, pb, nb, px, nx, rtol, maxit, C.byref(its), C.byref(rel)),
                    (FEM_OK, FEM_NOT_CONVERGED))
        return its.value, rel.value, rc == FEM_OK
