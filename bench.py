"""Benchmark: GMG-preconditioned CG solve of BASELINE.json configs[1] (C2) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C2]

One step = one complete solve (operator applies, Chebyshev
smoothing, transfers, coarse solve, PCG vector work) from x = 0 to ||r|| <= 1e-10 ||b||,
with the right-hand side already resident in HBM.  value = DoFs solved per second
over all ranks; ms_per_step = time to solution.  The dominant kernel (the
finest-level operator apply) is timed live with CUDA events on the library's
stream (fem_options.profile) and reported against the HBM roofline.

--impl reference times the CPU oracle (oracle/, the "reference" of this tier) on
the host cores: warm-up runs one full oracle solve (iteration count), each timed
step is one oracle PCG iteration; value = n_dofs / (t_iteration * iterations).
Multi-GPU (torchrun, one process per GPU): the mesh is split into z-slabs, one
C2-sized slab (32x32x32 cells) per GPU on the box [0,1]^2 x [0,N] (weak scaling);
libfem exchanges ghost planes with NCCL send/recv and all-reduces the PCG dot
products; value = global DoFs / max-over-ranks time.
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
METRIC = "GMG-CG solve throughput (DoFs solved per second; ms_per_step = time to solution)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="C2")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--rtol", type=float, default=1e-10)
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
    table on deformed meshes (6 doubles per quadrature point per cell)."""
    n_cells = int(np.prod(w.cells))
    geo = 48 * (w.degree + 1) ** 3 * n_cells if w.deform_eps else 0
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


def cpu_baseline(w, rtol):
    """The oracle as it stands: one full PCG solve of the same workload (setup excluded)."""
    mg, b = oracle_solver(w)
    t0 = time.perf_counter()
    _, its, rr = mg.pcg(b, tol=rtol)
    t = time.perf_counter() - t0
    n = mg.fine.n_dofs
    return {"value": n / t, "unit": "DoF/s", "cores": cpu_threads(), "kind": "oracle",
            "sample": f"one full oracle PCG solve of {w.name} ({its} iterations, relres {rr:.2e}), "
                      f"setup (geometry, lambda estimates, coarse Cholesky) excluded",
            "seconds": t}


# ---------------------------------------------------------------- reference arm
def run_reference(args, w):
    rank, world, _ = dist_env()
    if world > 1 and rank != 0:
        return
    from oracle import multigrid as omg
    mg, b = oracle_solver(w)
    n = mg.fine.n_dofs
    A = mg.fine.apply
    # warm-up: one complete solve gives the oracle's own iteration count
    _, its, rr = mg.pcg(b, tol=args.rtol)
    for _ in range(max(args.warmup - 1, 0)):
        mg.vcycle(b)
    # timed steps: one PCG iteration each (apply, two dots, updates, V-cycle)
    x = np.zeros_like(b)
    r = b.copy()
    z = mg.vcycle(r)
    p = z.copy()
    rz = r @ z
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        q = A(p)
        alpha = rz / (p @ q)
        x += alpha * p
        r -= alpha * q
        _ = np.linalg.norm(r)
        z = mg.vcycle(r)
        rz_new = r @ z
        p = z + (rz_new / rz) * p
        rz = rz_new
        times.append(time.perf_counter() - t0)
    t_iter = sum(times) / len(times)
    t_solve = t_iter * its
    value = n / t_solve
    line = {
        "impl": "reference", "metric": METRIC,
        "value": value, "unit": "DoF/s", "n_gpus": 0, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t_solve * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic", "config": {"workload": workload_desc(w), "n_dofs": n,
                                                         "rtol": args.rtol, "iterations": its},
        "cpu_baseline": {"value": value, "unit": "DoF/s", "cores": cpu_threads(), "kind": "oracle",
                         "sample": f"each step = one oracle PCG iteration on the full {w.name} problem; "
                                   f"value = n_dofs / (mean iteration time x {its} iterations)"},
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
        # weak scaling: one C2-sized z-slab per GPU, the box stretched to [0,1]^2 x [0,N]
        # so cells stay cubic; NCCL halo exchange + all-reduced dots
        import torch.distributed as dist
        cells = (w.cells[0], w.cells[1], w.cells[2] * world)
        hi = (w.hi[0], w.hi[1], w.hi[2] * world)
        obj = [fem.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        mp = dict(rank=rank, nranks=world, nccl_id=obj[0])
    F = fem.Fem(cells, w.degree, w.method, deform_eps=w.deform_eps, bc=w.bc, hi=hi,
                penalty_factor=w.penalty_factor, stream=stream, profile=True, **mp)
    n = F.n_local
    b = torch.zeros(n, dtype=torch.float64, device="cuda")
    if w.rhs == "manufactured":
        F.fem_rhs(b)
    else:
        xs = torch.from_numpy(fem_inputs.uniform_pm1(w.seed, n, F.first_global)).cuda()
        F.fem_apply(xs, b)
        del xs
        b[constrained_mask(w, n, cells, F.first_global)] = 0.0     # reading R15: b = A x_seed with Dirichlet rows zeroed
    x = torch.zeros_like(b)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")   # 256 MiB > L2

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

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
    t_ms = sum(step_ms)
    apply_ms, apply_launches = F.fem_profile_read(reset=True)
    if world > 1:
        import torch.distributed as dist
        tt = torch.tensor([t_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_ms = tt.item()
    value = F.n_global * args.steps / (t_ms * 1e-3)

    # end to end through the C ABI with host buffers (copies inside the timed region)
    bh = b.cpu().pin_memory()
    xh = torch.zeros(n, dtype=torch.float64).pin_memory()
    F.cg_solve(bh, xh, rtol=args.rtol)
    torch.cuda.synchronize()
    e2e_t = []
    for i in range(max(1, min(args.steps, 3))):
        flush.fill_(float(i))
        xh.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        F.cg_solve(bh, xh, rtol=args.rtol)
        e2e_t.append(time.perf_counter() - t0)
    e2e_s = sum(e2e_t) / len(e2e_t)
    if world > 1:
        import torch.distributed as dist
        tt = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_s = tt.item()
    e2e_value = F.n_global / e2e_s

    hbm, hbm_src = peaks()
    bytes_per_launch = algorithmic_apply_bytes(w, n)
    avg_apply_s = apply_ms * 1e-3 / max(apply_launches, 1)
    achieved = bytes_per_launch / avg_apply_s / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            entry = json.load(f).get(w.name)
        traffic = entry["bytes_per_launch"] if entry else None
    line = {
        "metric": METRIC,
        "value": value, "unit": "DoF/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t_ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_desc(w), "n_dofs": n, "rtol": args.rtol, "iterations": its,
                   "l2": "flushed between steps (256 MiB write, outside the per-step events)",
                   "n_dofs_global": F.n_global, "cells": list(cells), "box_hi": list(hi),
                   "parallelism": "single GPU" if world == 1 else
                   f"{world} z-slabs (NCCL halo exchange + all-reduce), one C2-sized slab per GPU",
                   "step_ms": [round(s, 4) for s in step_ms]},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                     "frac": achieved / hbm, "traffic": traffic,
                     "kernel": "finest-level operator apply (cg_apply_kernel for CG Q4 deformed); timed on the PCG apply q = A p of every iteration",
                     "algorithmic_bytes_per_launch": bytes_per_launch,
                     "avg_launch_us": avg_apply_s * 1e6, "launches": apply_launches,
                     "peak_source": hbm_src},
        "apply": {"dofs_per_s": n / avg_apply_s,
                  "equivalent_dofs_per_s": int(np.prod(w.cells)) * w.degree ** 3 / avg_apply_s},
        "clocks": clk,
        "e2e": {"value": e2e_value, "unit": "DoF/s", "h2d_bytes_per_step": 16 * n,
                "d2h_bytes_per_step": 8 * n},
        "gpu_launches": launches,
    }
    if rank == 0 and not args.no_cpu_baseline and world == 1:
        line["cpu_baseline"] = cpu_baseline(w, args.rtol)
        line["cpu_baseline"].pop("seconds", None)
    if rank == 0:
        print(json.dumps(line), flush=True)
    F.close()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def main():
    args = parse()
    w = fem_inputs.CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, w)
    else:
        run_ours(args, w)


if __name__ == "__main__":
    main()
