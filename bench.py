"""Benchmark: BASELINE.json's headline (configs[3] = C4, the largest single-GPU config).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C4]

One step = one complete GMG-CG solve (operator applies with the
fused Chebyshev smoother, transfers, coarse solve, PCG vector work) of C4 -- CG Q4 on a
Cartesian 128^3 mesh (135,005,697 DoFs), b = A x_7 with the Dirichlet rows zeroed
(reading R15) -- from x = 0 to ||r|| <= 1e-10 ||b||, with b resident in HBM.
value = DoFs solved per second over all ranks; ms_per_step = time to solution.  The
dominant kernel (the finest-level operator apply, kernels_stencil.cu K1t) is timed live
with CUDA events on the library's stream (fem_options.profile) on the PCG apply q = A p
of every iteration and reported against the measured HBM peak (algorithmic 16 B/DoF)
and, as an extra key, against the measured FP64 peak (algorithmic 7 banded sweeps,
2 (k+2) flop per DoF each).  `apply` adds the standalone y = A x_7 throughput
(actual and equivalent DoF/s).

--impl reference times the CPU oracle (oracle/, the reference of this tier) on the
host cores; each step is one complete oracle GMG-CG solve of the same recipe on a
bounded sample mesh (C4 recipe at 16^3 cells, 274,625 DoFs; setup untimed), value =
sample DoFs / step time.
--gpus N > 1 without torchrun re-launches itself under torch.distributed.run (one
process per GPU, 127.0.0.1 rendezvous).  Multi-GPU = strong scaling of the same C4
mesh split into z-slabs: NCCL halo exchange + all-reduced dots;
value = global DoFs / max-over-ranks time to solution.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import fem_inputs  # noqa: E402

FALLBACK_HBM_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback
METRIC = "FP64 operator-apply DoFs/s and GMG-CG time-to-solution; % of HBM roofline"   # BASELINE.json
FP64_PEAK_TFLOPS = 36.794   # profiles/fp64_peak.json (tools/fp64_peak.cu, measured on this pool's B200)
REF_SAMPLE_CELLS = (16, 16, 16)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="C4")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--rtol", type=float, default=1e-10)
    ap.add_argument("--no-hdg", action="store_true", help="skip the N4 HDG operator measurement")
    ap.add_argument("--others", default="C2,C3,C5",
                    help="single GPU: also time these configs' solves and applies (extra key other_configs)")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def workload_desc(w):
    return (f"{w.name}: {'CG' if w.method == fem_inputs.CG else 'SIPG'} Q{w.degree} "
            f"{'deformed (eps=%g)' % w.deform_eps if w.deform_eps else 'Cartesian'} "
            f"{w.cells[0]}x{w.cells[1]}x{w.cells[2]} on [0,1]^3, Dirichlet, "
            f"{'manufactured u=prod sin(pi x_d)' if w.rhs == 'manufactured' else 'b = A x_seed%d' % w.seed}")


def algorithmic_apply_bytes(w, n_dofs):
    """read x once + write y once (16 B/DoF) plus the streamed geometry
    table on deformed meshes (6 doubles per quadrature point per cell) and, for SIPG on
    deformed meshes, the face records (7 doubles per face quadrature point)."""
    n_cells = int(np.prod(w.cells))
    geo = 48 * (w.degree + 1) ** 3 * n_cells if w.deform_eps else 0
    if w.deform_eps and w.method == fem_inputs.SIPG:
        nx, ny, nz = w.cells
        n_faces = (nx + 1) * ny * nz + nx * (ny + 1) * nz + nx * ny * (nz + 1)
        geo += 56 * (w.degree + 1) ** 2 * n_faces
    return 16 * n_dofs + geo


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled DURING the timed region:
    NVML polled every 2 ms from a thread (the timed region is tens of ms), with
    nvidia-smi as the fallback when NVML is unavailable."""
    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"))

    def __init__(self, local_index):
        self.local, self.samples, self.max_mhz, self.stop_flag = local_index, [], None, False
        self.nv = self.handle = None
        try:
            import pynvml as nv
            import torch
            nv.nvmlInit()
            try:
                uuid = str(torch.cuda.get_device_properties(local_index).uuid)
                self.handle = nv.nvmlDeviceGetHandleByUUID(uuid if uuid.startswith("GPU-") else "GPU-" + uuid)
            except Exception:
                self.handle = nv.nvmlDeviceGetHandleByIndex(local_index)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(self.handle, nv.NVML_CLOCK_SM)
            self.nv = nv
        except Exception:
            self.nv = None

    def _poll(self):
        nv = self.nv
        while not self.stop_flag:
            try:
                mhz = nv.nvmlDeviceGetClockInfo(self.handle, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.handle)
                self.samples.append((mhz, rs))
            except Exception:
                pass
            time.sleep(0.002)

    def start(self):
        self.samples.clear()
        self.stop_flag = False
        if self.nv is not None:
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
        else:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.local}", "--query-gpu=clocks.sm,clocks.max.sm,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)

    def stop(self):
        self.stop_flag = True
        names = [n for n, _ in self.REASONS]
        if self.nv is not None:
            self.t.join(timeout=1)
            sm = [m for m, _ in self.samples]
            bits = [(n, getattr(self.nv, c, 0)) for n, c in self.REASONS]
            reasons = sorted({n for _, rs in self.samples for n, b in bits if b and rs & b})
            mx = self.max_mhz
            src = "nvml (2 ms polling)"
        else:
            self.proc.terminate()
            out = self.proc.communicate(timeout=5)[0]
            rows = [[p.strip() for p in ln.split(",")] for ln in out.splitlines() if ln.count(",") == 5]
            sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
            mx = max((float(r[1]) for r in rows if r[1].replace(".", "").isdigit()), default=None)
            reasons = sorted({names[i] for r in rows for i in range(4) if r[2 + i] == "Active"})
            src = "nvidia-smi (20 ms)"
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": reasons, "samples": len(sm), "source": src}


def cpu_threads():
    try:
        from threadpoolctl import threadpool_info
        return max((i.get("num_threads", 1) for i in threadpool_info()), default=os.cpu_count())
    except Exception:
        return os.cpu_count()


def oracle_solver(w):
    from oracle import multigrid as omg, problem as oprob
    from oracle.mesh import Mesh
    m = Mesh(w.cells, w.degree, eps=w.deform_eps, bc=w.bc)
    mg = omg.Multigrid(m, w.method, penalty_factor=w.penalty_factor)
    if w.rhs == "manufactured":
        b = oprob.rhs(m, w.method)
    else:
        x7 = fem_inputs.uniform_pm1(w.seed, mg.fine.n_dofs)
        b = mg.fine.apply(x7)
        b[~mg.fine.free] = 0.0
    return mg, b


def oracle_sample(w):
    """The bounded CPU sample of a workload: the same recipe on REF_SAMPLE_CELLS when the
    full mesh is larger (the oracle's cost per DoF does not depend on the mesh size)."""
    if int(np.prod(w.cells)) <= int(np.prod(REF_SAMPLE_CELLS)):
        return w, "the full workload"
    ws = fem_inputs.scaled(w, REF_SAMPLE_CELLS)
    return ws, (f"the {w.name} recipe (same method, degree, deformation, boundary conditions, "
                f"right-hand side) on {REF_SAMPLE_CELLS[0]}x{REF_SAMPLE_CELLS[1]}x{REF_SAMPLE_CELLS[2]} cells")


def cpu_baseline(w, rtol):
    """The oracle as it stands: one full PCG solve of the bounded sample (setup excluded)."""
    ws, what = oracle_sample(w)
    mg, b = oracle_solver(ws)
    t0 = time.perf_counter()
    _, its, rr = mg.pcg(b, tol=rtol)
    t = time.perf_counter() - t0
    n = mg.fine.n_dofs
    return {"value": n / t, "unit": "DoF/s", "cores": cpu_threads(), "kind": "oracle",
            "sample": f"one full oracle GMG-PCG solve of {what} ({n} DoFs, {its} iterations, "
                      f"relres {rr:.2e}); setup (geometry, lambda estimates, coarse Cholesky) excluded",
            "seconds": t}


# ---------------------------------------------------------------- reference arm
def run_reference(args, w):
    rank, world, _ = dist_env()
    if world > 1 and rank != 0:
        return
    ws, what = oracle_sample(w)
    t_setup = time.perf_counter()
    mg, b = oracle_solver(ws)
    t_setup = time.perf_counter() - t_setup
    n = mg.fine.n_dofs
    its = 0
    for _ in range(args.warmup):
        _, its, rr = mg.pcg(b, tol=args.rtol)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        _, its, rr = mg.pcg(b, tol=args.rtol)
        times.append(time.perf_counter() - t0)
        assert rr <= args.rtol
    t_step = sum(times) / len(times)
    value = n / t_step
    line = {
        "impl": "reference", "metric": METRIC,
        "value": value, "unit": "DoF/s", "n_gpus": 0, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t_step * 1e3, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_desc(w), "n_dofs_global": w.n_dofs(), "n_dofs_local": w.n_dofs(),
                   "rtol": args.rtol, "iterations": its, "cells": list(w.cells),
                   "l2": "n/a (CPU oracle)", "parallelism": "CPU oracle (numpy, host cores)",
                   "setup_s": round(t_setup, 3), "residual_history": None, "err_vs_x7": None,
                   "sample_cells": list(ws.cells), "sample_n_dofs": n,
                   "step_ms": [round(t * 1e3, 4) for t in times]},
        "cpu_baseline": {"value": value, "unit": "DoF/s", "cores": cpu_threads(), "kind": "oracle",
                         "sample": f"each step = one full oracle GMG-PCG solve of {what} ({n} DoFs, "
                                   f"{its} iterations, setup untimed); value = sample DoFs / mean step time"},
        "e2e": {"value": value, "unit": "DoF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def constrained_mask(w, n, cells, first=0):
    """Dirichlet-constrained CG nodes of the owned slice (input preparation only; index arithmetic)."""
    import torch
    k = w.degree
    nn = [k * c + 1 for c in cells]
    i = torch.arange(first, first + n, device="cuda")
    g = [i % nn[0], (i // nn[0]) % nn[1], i // (nn[0] * nn[1])]
    m = torch.zeros(n, dtype=torch.bool, device="cuda")
    for d in range(3):
        if w.bc[2 * d] == fem_inputs.DIRICHLET:
            m |= g[d] == 0
        if w.bc[2 * d + 1] == fem_inputs.DIRICHLET:
            m |= g[d] == nn[d] - 1
    return m


def apply_flops_per_dof(w):
    """Algorithmic FP64 flops of one apply per DoF: Cartesian CG = 7 banded 1-D sweeps of the
    assembled Kronecker sum (App. B), k + 2 FMA per node each (vertex rows 2k+1 entries,
    interior rows k+1); other paths: SURVEY §8d estimates are not used for the roofline."""
    if w.method == fem_inputs.CG and not w.deform_eps:
        return 2 * 7 * (w.degree + 2)
    return None


# ---------------------------------------------------------------- other configs
def other_configs(names, rtol, reps=5):
    """BASELINE.json's other solve configs measured in the same run (single GPU): time to
    solution (median of `reps` solves from x = 0, CUDA events, L2 flushed between them),
    iterations, and the finest-level apply (20 back to back between two events; the
    algorithmic bytes of algorithmic_apply_bytes)."""
    import torch
    from paper_1611_03029_b200 import fem
    hbm, _ = peaks()
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    out = {}
    for name in names:
        w = fem_inputs.CONFIGS[name]
        t0 = time.perf_counter()
        F = fem.Fem(w.cells, w.degree, w.method, deform_eps=w.deform_eps, bc=w.bc,
                    penalty_factor=w.penalty_factor)
        torch.cuda.synchronize()
        setup = time.perf_counter() - t0
        n = F.n_local
        b = torch.zeros(n, dtype=torch.float64, device="cuda")
        F.fem_rhs(b)
        x = torch.zeros_like(b)
        F.cg_solve(b, x, rtol=rtol)
        ts, its = [], 0
        for i in range(reps):
            flush.fill_(float(i))
            x.zero_()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            its, rr, ok = F.cg_solve(b, x, rtol=rtol)
            e.record()
            torch.cuda.synchronize()
            assert ok and rr <= rtol
            ts.append(s.elapsed_time(e))
        xa = torch.from_numpy(fem_inputs.uniform_pm1(w.seed, n)).cuda()
        ya = torch.empty_like(xa)
        F.fem_apply(xa, ya)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        s.record()
        for _ in range(20):
            F.fem_apply(xa, ya)
        e.record()
        torch.cuda.synchronize()
        t_apply = s.elapsed_time(e) * 1e-3 / 20
        t_solve = statistics.median(ts) * 1e-3
        n_cells = int(np.prod(w.cells))
        out[name] = {"workload": workload_desc(w), "n_dofs": n, "iterations": its,
                     "time_to_solution_ms": t_solve * 1e3, "dofs_per_s": n / t_solve,
                     "apply_us": t_apply * 1e6, "apply_dofs_per_s": n / t_apply,
                     "apply_equivalent_dofs_per_s": n_cells * w.degree ** 3 / t_apply,
                     "apply_hbm_frac": algorithmic_apply_bytes(w, n) / t_apply / 1e9 / hbm,
                     "setup_s": round(setup, 3), "solve_ms_samples": [round(t, 4) for t in ts]}
        F.close()
        del b, x, xa, ya
        torch.cuda.empty_cache()
    return out


def hdg_flops_per_cell(k):
    """Algorithmic FMA x 2 of one HDG trace apply per cell (csrc/hdg.cu): face masses in and out
    12 + 12 n^3, t-tensor 6 n^3, fast-diagonalization sweeps 6 n^4, face-layer reductions 6 n^3."""
    n = k + 1
    return 2 * (6 * n ** 4 + 36 * n ** 3)


def hdg_mixed_flops_per_cell(k):
    """Mixed apply per cell: per direction 3 n^4 (slot-d operators) + 4 n^4 (two tangential mass
    sweeps of two fields): 21 n^4 FMA."""
    return 2 * 21 * (k + 1) ** 4


def hdg_config(cells=(32, 32, 32), k=4, rtol=1e-10, reps=20, solve=True, deform_eps=0.0):
    """HDG Q_k on the C3 mesh (Cartesian, Dirichlet, manufactured u):
    trace matrix-free and mixed matrix-free applies (reps back to back between CUDA events) with
    their FP64 and HBM roofline fractions, and the Jacobi-PCG trace solve (iterations, time)."""
    import torch
    from paper_1611_03029_b200 import fem
    hbm, _ = peaks()
    H = fem.Hdg(cells, k, deform_eps=deform_eps)
    nt, nc = H.n_trace, H.n_cells
    x = torch.from_numpy(fem_inputs.uniform_pm1(0, nt)).cuda()
    y = torch.empty_like(x)

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(reps):
            fn()
        e.record()
        torch.cuda.synchronize()
        return s.elapsed_time(e) * 1e-3 / reps

    t_tr = timed(lambda: H.hdg_apply(x, y))
    m = (k + 1) ** 3
    if deform_eps:   # the paper's design: S^-1 stored per cell (read once per apply); no mixed form
        H.close()
        stored = nc * m * m * 8
        return {"workload": f"N4: HDG Q{k} deformed (eps={deform_eps}) {cells[0]}x{cells[1]}x{cells[2]}, Dirichlet, "
                            f"tau = 5, local inverse stored per cell (the paper's design)",
                "n_trace_dofs": nt, "n_cells": nc, "trace_apply_us": t_tr * 1e6, "trace_dofs_per_s": nt / t_tr,
                "trace_equivalent_dofs_per_s": nc * k ** 3 / t_tr,
                "trace_hbm_frac": (16.0 * nt + stored) / t_tr / 1e9 / hbm, "stored_inverse_bytes": stored}
    qu = torch.from_numpy(fem_inputs.uniform_pm1(1, 4 * nc * m)).cuda()
    yq = torch.empty_like(qu)
    t_mx = timed(lambda: H.hdg_mixed_apply(qu, yq))
    its, rr, ok, ms = 0, None, None, None
    if solve:
        b = torch.zeros(nt, dtype=torch.float64, device="cuda")
        H.hdg_rhs(b)
        lam = torch.zeros_like(b)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        its, rr, ok = H.hdg_cg_solve(b, lam, rtol=rtol)
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e)
    eq = nc * k ** 3
    fl_tr, fl_mx = hdg_flops_per_cell(k) * nc, hdg_mixed_flops_per_cell(k) * nc
    out = {"workload": f"N4: HDG Q{k} Cartesian {cells[0]}x{cells[1]}x{cells[2]} on [0,1]^3, Dirichlet, tau = 5",
           "n_trace_dofs": nt, "n_cells": nc,
           "trace_apply_us": t_tr * 1e6, "trace_dofs_per_s": nt / t_tr, "trace_equivalent_dofs_per_s": eq / t_tr,
           "trace_fp64_frac": fl_tr / t_tr / 1e12 / FP64_PEAK_TFLOPS,
           "trace_hbm_frac": 16.0 * nt / t_tr / 1e9 / hbm,
           "mixed_apply_us": t_mx * 1e6, "mixed_dofs_per_s": 4 * nc * m / t_mx, "mixed_equivalent_dofs_per_s": eq / t_mx,
           "mixed_fp64_frac": fl_mx / t_mx / 1e12 / FP64_PEAK_TFLOPS,
           "mixed_hbm_frac": 64.0 * nc * m / t_mx / 1e9 / hbm,
           "jacobi_pcg": {"iterations": its, "relres": rr, "converged": ok, "ms": ms},
           "flops_per_cell": {"trace": hdg_flops_per_cell(k), "mixed": hdg_mixed_flops_per_cell(k)}}
    H.close()
    return out


# ---------------------------------------------------------------- our arm
def run_ours(args, w):
    import torch
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_1611_03029_b200 import fem

    stream = torch.cuda.current_stream()
    cells, hi, mp = w.cells, w.hi, {}
    if world > 1:
        # strong scaling: the same mesh in z-slabs, NCCL halo exchange + all-reduced dots
        import torch.distributed as dist
        obj = [fem.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        mp = dict(rank=rank, nranks=world, nccl_id=obj[0])
    t_setup = time.perf_counter()
    F = fem.Fem(cells, w.degree, w.method, deform_eps=w.deform_eps, bc=w.bc, hi=hi,
                penalty_factor=w.penalty_factor, stream=stream, profile=True, **mp)
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t_setup
    n = F.n_local
    b = torch.zeros(n, dtype=torch.float64, device="cuda")
    xs = None
    if w.rhs == "manufactured":
        F.fem_rhs(b)
    else:
        xs = torch.from_numpy(fem_inputs.uniform_pm1(w.seed, n, F.first_global)).cuda()
        F.fem_apply(xs, b)
        b[constrained_mask(w, n, cells, F.first_global)] = 0.0     # reading R15: b = A x_seed with Dirichlet rows zeroed
    x = torch.zeros_like(b)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")   # 256 MiB > L2

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    def max_over_ranks(v):
        if world == 1:
            return v
        import torch.distributed as dist
        tt = torch.tensor([v], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        return tt.item()

    clocks = ClockSampler(local)
    its = 0
    for _ in range(args.warmup):
        x.zero_()
        its, rr, ok = F.cg_solve(b, x, rtol=args.rtol)
        assert ok, "warm-up solve did not converge"
    F.fem_profile_read(reset=True)
    launches0 = fem.kernel_launches()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    barrier()
    torch.cuda.synchronize()
    clocks.start()
    for i in range(args.steps):
        flush.fill_(float(i))                       # evict L2 between steps (not timed)
        x.zero_()
        starts[i].record(stream)
        its, rr, ok = F.cg_solve(b, x, rtol=args.rtol)
        ends[i].record(stream)
        assert ok and rr <= args.rtol
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    launches = fem.kernel_launches() - launches0
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    t_ms = max_over_ranks(sum(step_ms))
    apply_ms, apply_launches = F.fem_profile_read(reset=True)
    value = F.n_global * args.steps / (t_ms * 1e-3)
    hist = F.cg_history()
    err_x7 = None
    if xs is not None:   # R15 pin: the solve returns x_7 on the free DoFs
        fm = ~constrained_mask(w, n, cells, F.first_global)
        err_x7 = ((x - xs)[fm].norm() / xs[fm].norm()).item()

    # the dominant kernel of the step: the finest-level Chebyshev step (fused into the K1t apply
    # on C4: MODE 1), timed live with CUDA events on the library's stream over a second timed
    # pass of the same solves (profile mode 2: an event pair around every finest smoother step)
    F.fem_profile_mode(2)
    x.zero_()
    F.cg_solve(b, x, rtol=args.rtol)          # re-captures the PCG graphs with the event nodes
    F.fem_profile_read_bytes(reset=True)
    step_ms2 = []
    for i in range(args.steps):
        flush.fill_(float(i))
        x.zero_()
        s2, e2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s2.record(stream)
        F.cg_solve(b, x, rtol=args.rtol)
        e2.record(stream)
        torch.cuda.synchronize()
        step_ms2.append(s2.elapsed_time(e2))
    live_ms, live_launches, live_bytes = F.fem_profile_read_bytes(reset=True)
    live_ms = max_over_ranks(live_ms)
    F.fem_profile_mode(1)

    # standalone apply y = A x (the north_star's apply DoF/s), inputs resident, > L2
    xa = xs if xs is not None else b
    ya = torch.empty_like(b)
    F.fem_apply(xa, ya)
    F.fem_profile_read(reset=True)
    sa, ea = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    barrier()
    torch.cuda.synchronize()
    sa.record(stream)
    for _ in range(reps):
        F.fem_apply(xa, ya)
    ea.record(stream)
    torch.cuda.synchronize()
    apply_s = max_over_ranks(sa.elapsed_time(ea) * 1e-3 / reps)
    F.fem_profile_read(reset=True)
    del ya

    # the finest-level Chebyshev smoother (R7): the launches that dominate the solve (the fused
    # step of K1t MODE 1 on C4); one mg_smooth from x != 0 = p = 5 steps, the first without
    # x_old: algorithmic bytes read x, (x_old), b, write x_new = (24 + 4 x 32) / 5 B per DoF
    smoother = None
    if world == 1:
        xsm = torch.zeros_like(b)
        fine = F.n_levels - 1
        F.mg_smooth(fine, b, xsm, False)
        smr = 5
        torch.cuda.synchronize()
        ss, es = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ss.record(stream)
        for _ in range(smr):
            F.mg_smooth(fine, b, xsm, False)
        es.record(stream)
        torch.cuda.synchronize()
        step_s = ss.elapsed_time(es) * 1e-3 / (5 * smr)
        sm_bytes = (24 + 4 * 32) / 5 * n
        smoother = {"step_us": step_s * 1e6, "algorithmic_bytes_per_step": sm_bytes,
                    "achieved_gbs": sm_bytes / step_s / 1e9,
                    "note": "finest-level Chebyshev step (fused into the operator apply on Cartesian CG levels): "
                            "mg_smooth from x != 0, 5 steps per call, CUDA events around 5 calls"}
        F.fem_profile_read(reset=True)
        del xsm

    # finest-level transfers (R8; node-grid kernels on C4): x_f += P x_c reads x_c, reads and writes
    # x_f (16 B per fine + 8 B per coarse DoF); r_c = P^T (b - A x) reads two fine vectors, writes r_c
    transfers = None
    if world == 1 and w.method == fem_inputs.CG and F.n_levels > 1:
        fine = F.n_levels - 1
        ncd = F.level_info(fine - 1)[0]
        xc = torch.from_numpy(fem_inputs.uniform_pm1(3, ncd)).cuda()
        rc = torch.zeros_like(xc)
        xf = b.clone()

        def timed_us(fn, reps=10):
            fn()
            torch.cuda.synchronize()
            s_, e_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s_.record(stream)
            for _ in range(reps):
                fn()
            e_.record(stream)
            torch.cuda.synchronize()
            return s_.elapsed_time(e_) * 1e3 / reps

        p_us = timed_us(lambda: F.mg_prolongate_add(fine, xc, xf))
        r_us = timed_us(lambda: F.mg_restrict(fine, b, rc))
        transfers = {"prolongate_add_us": p_us, "prolongate_algorithmic_bytes": 16 * n + 8 * ncd,
                     "restrict_us": r_us, "restrict_algorithmic_bytes": 8 * n + 8 * ncd,
                     "note": "finest level, standalone; the restriction here reads one fine vector (P^T b) and "
                             "includes the zero fill of the coarse vector"}
        F.fem_profile_read(reset=True)
        del xc, rc, xf

    # end to end through the C ABI with host buffers (copies inside the timed region)
    bh = b.cpu().pin_memory()
    xh = torch.zeros(n, dtype=torch.float64).pin_memory()
    F.cg_solve_zero(bh, xh, rtol=args.rtol)     # zero start: x is output only, not uploaded
    torch.cuda.synchronize()
    e2e_t = []
    for i in range(max(1, min(args.steps, 3))):
        flush.fill_(float(i))
        xh.zero_()
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        F.cg_solve_zero(bh, xh, rtol=args.rtol)
        e2e_t.append(time.perf_counter() - t0)
    e2e_s = max_over_ranks(sum(e2e_t) / len(e2e_t))
    e2e_value = F.n_global / e2e_s

    hbm, hbm_src = peaks()
    sm_avg_s = live_ms * 1e-3 / max(live_launches, 1)
    sm_bpl = live_bytes / max(live_launches, 1)
    sm_traffic = None
    try:
        sm_traffic = json.load(open(os.path.join(ROOT, "profiles", "traffic.json"))).get(w.name + "_smoother", {}).get("bytes_per_launch")
    except (OSError, ValueError):
        pass
    smoother_roofline = {
        "bound": "hbm", "achieved": sm_bpl / sm_avg_s / 1e9, "peak": hbm, "unit": "GB/s",
        "frac": sm_bpl / sm_avg_s / 1e9 / hbm, "traffic": sm_traffic,
        "kernel": "finest-level Chebyshev smoothing step (dominant: fused into the K1t apply, "
                  "cg_stencil2_kernel<4,1>, on C4); timed on every finest step of a second timed pass",
        "algorithmic_bytes_per_launch": sm_bpl, "avg_launch_us": sm_avg_s * 1e6, "launches": live_launches,
        "timed_pass_ms_per_step": statistics.mean(step_ms2) if step_ms2 else None,
        "peak_source": hbm_src}
    if smoother:
        smoother["hbm_frac"] = smoother["achieved_gbs"] / hbm
    if transfers:
        transfers["prolongate_hbm_frac"] = transfers["prolongate_algorithmic_bytes"] / (transfers["prolongate_add_us"] * 1e-6) / 1e9 / hbm
        transfers["restrict_hbm_frac"] = transfers["restrict_algorithmic_bytes"] / (transfers["restrict_us"] * 1e-6) / 1e9 / hbm
    bytes_per_launch = algorithmic_apply_bytes(w, n)
    avg_apply_s = apply_ms * 1e-3 / max(apply_launches, 1)
    achieved = bytes_per_launch / avg_apply_s / 1e9
    fpd = apply_flops_per_dof(w)
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            entry = json.load(f).get(w.name)
        traffic = entry["bytes_per_launch"] if entry else None
    n_cells = int(np.prod(w.cells))
    kern = ("cg_stencil2_kernel<4,0> (K1t, atomic-free assembled Kronecker stencil)"
            if w.method == fem_inputs.CG and not w.deform_eps else
            "cg_apply_kernel (K1)" if w.method == fem_inputs.CG else "dg kernels (K2/K3)")
    line = {
        "metric": METRIC,
        "value": value, "unit": "DoF/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t_ms / args.steps, "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_desc(w), "n_dofs_global": F.n_global, "n_dofs_local": n,
                   "rtol": args.rtol, "iterations": its, "cells": list(cells),
                   "l2": "flushed between steps (256 MiB write, outside the per-step events); vectors 1.08 GB each > L2",
                   "parallelism": "single GPU" if world == 1 else
                   f"{world} z-slabs of the same mesh (NCCL halo exchange + all-reduce), strong scaling",
                   "setup_s": round(t_setup, 3),
                   "residual_history": [float("%.4e" % h) for h in hist],
                   "err_vs_x7": err_x7,
                   "sample_cells": list(cells), "sample_n_dofs": F.n_global,
                   "step_ms": [round(s, 4) for s in step_ms]},
        "roofline": smoother_roofline,
        "apply_roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                           "frac": achieved / hbm, "traffic": traffic,
                           "kernel": f"finest-level operator apply, {kern}; timed on the PCG apply q = A p of every iteration",
                           "algorithmic_bytes_per_launch": bytes_per_launch,
                           "avg_launch_us": avg_apply_s * 1e6, "launches": apply_launches,
                           "peak_source": hbm_src},
        "apply": {"us": apply_s * 1e6, "dofs_per_s": F.n_global / apply_s,
                  "equivalent_dofs_per_s": n_cells * w.degree ** 3 / apply_s,
                  "hbm_frac": algorithmic_apply_bytes(w, F.n_global) / apply_s / 1e9 / hbm},
        "clocks": clk,
        "smoother": smoother,
        "transfers": transfers,
        "e2e": {"value": e2e_value, "unit": "DoF/s", "h2d_bytes_per_step": 8 * n,
                "d2h_bytes_per_step": 8 * n, "call": "cg_solve_zero(b host, x host): b uploaded, x downloaded"},
        "gpu_launches": launches,
    }
    if fpd:
        fl = fpd * n
        line["apply_roofline"]["fp64"] = {"algorithmic_flops_per_launch": fl,
                                          "achieved_tflops": fl / avg_apply_s / 1e12,
                                          "peak_tflops": FP64_PEAK_TFLOPS,
                                          "frac": fl / avg_apply_s / 1e12 / FP64_PEAK_TFLOPS,
                                          "peak_source": "profiles/fp64_peak.json (measured DFMA chains)"}
        # the fused step does the apply's flops (its epilogue adds ~5 per DoF, not counted)
        line["roofline"]["fp64"] = {"algorithmic_flops_per_launch": fl,
                                    "achieved_tflops": fl / sm_avg_s / 1e12,
                                    "peak_tflops": FP64_PEAK_TFLOPS,
                                    "frac": fl / sm_avg_s / 1e12 / FP64_PEAK_TFLOPS,
                                    "peak_source": "profiles/fp64_peak.json (measured DFMA chains)"}
        line["apply"]["fp64_frac"] = fpd * F.n_global / apply_s / 1e12 / FP64_PEAK_TFLOPS
    F.close()
    if world == 1 and args.others:
        del b, x, flush
        torch.cuda.empty_cache()
        line["other_configs"] = other_configs([c for c in args.others.split(",") if c != w.name], args.rtol)
        if not args.no_hdg:
            line["other_configs"]["N4_HDG"] = hdg_config(rtol=args.rtol)
            line["other_configs"]["N4_HDG_deformed"] = hdg_config(rtol=args.rtol, deform_eps=0.05, reps=5)
    if rank == 0 and not args.no_cpu_baseline and world == 1:
        line["cpu_baseline"] = cpu_baseline(w, args.rtol)
        line["cpu_baseline"].pop("seconds", None)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def respawn_under_torchrun(args):
    """--gpus N > 1 outside torchrun: one process per GPU via torch.distributed.run."""
    import random
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(random.randint(20000, 40000)),
           os.path.abspath(__file__)] + sys.argv[1:]
    os.execv(sys.executable, cmd)


def main():
    args = parse()
    w = fem_inputs.CONFIGS[args.config]
    _, world, _ = dist_env()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        respawn_under_torchrun(args)
    if args.impl == "ours" and world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        run_reference(args, w)
    else:
        run_ours(args, w)


if __name__ == "__main__":
    main()
