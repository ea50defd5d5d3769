// libfem C ABI (include/fem.h): setup, operator entry points, V-cycle, PCG.
//
// Host orchestration only: every arithmetic step on vectors runs in the kernels
// of kernels_cg.cu / kernels_dg.cu / kernels_mg.cu.  The host does the O(1)
// scalar work of the paper's algorithms: Chebyshev coefficients,
// the 15x15 Lanczos eigenvalue problem, the PCG stopping test
// (P:L1146-1148), and the tiny dense Cholesky factorisation of the coarse
// matrix (R9), which is assembled on the device by the level-0 operator.
#include <algorithm>
#include <array>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "internal.h"
#include "device_common.cuh"

namespace fem {

void launch_cg_apply(fem_ctx* h, const Level& L, const double* x, double* y, int64_t c0 = 0, int64_t c1 = -1);
void launch_cg_diagonal(fem_ctx* h, Level& L);
void launch_dg_apply(fem_ctx* h, const Level& L, const double* x, double* y, int64_t c0 = 0, int64_t c1 = -1);
void launch_dg_diagonal(fem_ctx* h, Level& L);
void launch_dg_face_geometry(fem_ctx* h, Level& L);

namespace {
thread_local std::string g_last_error;
std::atomic<int64_t> g_launches{0};
thread_local int64_t* g_capture_count = nullptr;   // set while a graph is captured
}  // namespace

void set_error(const std::string& msg) { g_last_error = msg; }
void count_launch(int n) {
  if (g_capture_count) *g_capture_count += n;
  else g_launches += n;
}
void smem_attr(const void* func, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> done;
  int dev = 0;
  FEM_CUDA_TRY(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  size_t& cur = done[{func, dev}];
  if (cur >= bytes) return;
  FEM_CUDA_TRY(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  cur = bytes;
}

void check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw Error{FEM_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e)};
}

namespace {

double* dalloc(int64_t n) {
  void* p = nullptr;
  FEM_CUDA_TRY(cudaMalloc(&p, sizeof(double) * std::max<int64_t>(n, 1)));
  return (double*)p;
}

void dfree(double*& p) {
  if (p) cudaFree(p);
  p = nullptr;
}

// level vectors: owned block plus ghosts, pointer at the owned block (internal.h)
// (cudaMemset runs on the legacy default stream, which is not ordered with a
// non-blocking user stream: wait for it before any kernel on h->stream can touch p)
double* valloc(const Level& L) {
  double* p = dalloc(L.n_store);
  FEM_CUDA_TRY(cudaMemset(p, 0, sizeof(double) * L.n_store));
  FEM_CUDA_TRY(cudaDeviceSynchronize());
  return p + L.own_off;
}

void vfree(const Level& L, double*& p) {
  if (p) cudaFree(p - L.own_off);
  p = nullptr;
}

// ---------------------------------------------------------------- profiling
cudaEvent_t new_event() {
  cudaEvent_t e;
  FEM_CUDA_TRY(cudaEventCreate(&e));
  return e;
}

void prof_begin(fem_ctx* h, bool finest, double bytes = 0.0) {
  if (!h->prof.on || !finest) return;
  if (h->prof.capturing) {
    // external record nodes: the events are really recorded on every replay, so
    // cudaEventElapsedTime works on them after the graph has run
    h->prof.cap->push_back({new_event(), new_event()});
    if (h->prof.capb) h->prof.capb->push_back(bytes);
    FEM_CUDA_TRY(cudaEventRecordWithFlags(h->prof.cap->back().first, h->stream, cudaEventRecordExternal));
    return;
  }
  if (h->prof.used + 2 > h->prof.ev.size()) {
    for (int i = 0; i < 64; ++i) {
      cudaEvent_t e;
      FEM_CUDA_TRY(cudaEventCreate(&e));
      h->prof.ev.push_back(e);
    }
  }
  FEM_CUDA_TRY(cudaEventRecord(h->prof.ev[h->prof.used], h->stream));
  if (h->prof.evb.size() < h->prof.ev.size() / 2) h->prof.evb.resize(h->prof.ev.size() / 2);
  h->prof.evb[h->prof.used / 2] = bytes;
}

void prof_end(fem_ctx* h, bool finest) {
  if (!h->prof.on || !finest) return;
  if (h->prof.capturing) {
    FEM_CUDA_TRY(cudaEventRecordWithFlags(h->prof.cap->back().second, h->stream, cudaEventRecordExternal));
    return;
  }
  FEM_CUDA_TRY(cudaEventRecord(h->prof.ev[h->prof.used + 1], h->stream));
  h->prof.used += 2;
  h->prof.launches += 1;
}

void prof_collect(fem_ctx* h) {
  if (!h->prof.on || h->prof.used == 0) return;
  FEM_CUDA_TRY(cudaStreamSynchronize(h->stream));
  for (size_t i = 0; i < h->prof.used; i += 2) {
    float ms = 0;
    FEM_CUDA_TRY(cudaEventElapsedTime(&ms, h->prof.ev[i], h->prof.ev[i + 1]));
    h->prof.ms += ms;
    h->prof.bytes += h->prof.evb[i / 2];
  }
  h->prof.used = 0;
}

// elapsed time of the event pairs of a graph that has completed (stream synchronised)
void prof_graph(fem_ctx* h, const std::vector<std::pair<cudaEvent_t, cudaEvent_t>>& ev,
                const std::vector<double>& evb) {
  if (!h->prof.on) return;
  for (size_t i = 0; i < ev.size(); ++i) {
    float ms = 0;
    FEM_CUDA_TRY(cudaEventElapsedTime(&ms, ev[i].first, ev[i].second));
    h->prof.ms += ms;
    h->prof.launches += 1;
    if (i < evb.size()) h->prof.bytes += evb[i];
  }
}

// ---------------------------------------------------------------- z-slab exchanges
// Message tags (they only matter to the in-process transport; NCCL pairs the
// single message per direction and neighbour pair by issue order).
enum { kTagCgImport = 1, kTagCgExport = 2, kTagDgToUpper = 3, kTagDgToLower = 4 };

}  // namespace

namespace {
void halo_import_on(fem_ctx* h, const Level& L, double* v, cudaStream_t stream);
void halo_export_send(fem_ctx* h, const Level& L, double* v, cudaStream_t stream);
}  // namespace

void halo_import(fem_ctx* h, const Level& L, double* v) { halo_import_on(h, L, v, h->stream); }

void halo_export_add(fem_ctx* h, const Level& L, double* v) {
  if (!L.dist || !h->comm || !is_cg(h)) return;
  halo_export_send(h, L, v, h->stream);
  if (L.ghost_lo >= 0) launch_add(h, v, L.halo, (int64_t)L.nn[0] * L.nn[1]);
}

namespace {
void halo_import_on(fem_ctx* h, const Level& L, double* v, cudaStream_t stream) {
  if (!L.dist || !h->comm) return;
  std::vector<Comm::Msg> snd, rcv;
  if (is_cg(h)) {
    // ghost plane k n[2] <- plane 0 of the rank above
    const int64_t plane = (int64_t)L.nn[0] * L.nn[1];
    if (L.ghost_lo >= 0) snd.push_back({L.ghost_lo, kTagCgImport, v, plane});
    if (L.ghost_hi >= 0) rcv.push_back({L.ghost_hi, kTagCgImport, v + (int64_t)h->k * L.n[2] * plane, plane});
  } else {
    const int64_t layer = (int64_t)L.n[0] * L.n[1] * (h->k + 1) * (h->k + 1) * (h->k + 1);
    if (L.ghost_lo >= 0) {
      snd.push_back({L.ghost_lo, kTagDgToUpper, v, layer});              // my bottom layer -> its top ghost
      rcv.push_back({L.ghost_lo, kTagDgToLower, v - layer, layer});      // its top layer -> my bottom ghost
    }
    if (L.ghost_hi >= 0) {
      snd.push_back({L.ghost_hi, kTagDgToLower, v + L.n_dofs - layer, layer});
      rcv.push_back({L.ghost_hi, kTagDgToUpper, v + L.n_dofs, layer});
    }
  }
  h->comm->exchange(snd, rcv, stream);
}

// CG: send the ghost node plane of v to the rank above, receive the one of the rank
// below into L.halo (the caller adds it into plane 0)
void halo_export_send(fem_ctx* h, const Level& L, double* v, cudaStream_t stream) {
  const int64_t plane = (int64_t)L.nn[0] * L.nn[1];
  std::vector<Comm::Msg> snd, rcv;
  if (L.ghost_hi >= 0) snd.push_back({L.ghost_hi, kTagCgExport, v + (int64_t)h->k * L.n[2] * plane, plane});
  if (L.ghost_lo >= 0) rcv.push_back({L.ghost_lo, kTagCgExport, L.halo, plane});
  h->comm->exchange(snd, rcv, stream);
}
}  // namespace

void allreduce(fem_ctx* h, double* p, int64_t n) {
  if (h->comm) h->comm->allreduce_sum(p, n, h->stream);
}

namespace {

// dot product of owned entries into h->scal[slot], summed over ranks on distributed levels
void dot(fem_ctx* h, const Level& L, const double* a, const double* b, int slot) {
  launch_dot(h, a, b, L.n_dofs, slot);
  if (L.dist) allreduce(h, h->scal + slot, 1);
}

// ---------------------------------------------------------------- operator
// y = A x on level L.  y is overwritten.  CG: constrained rows y_c = x_c.
// On a distributed level x must be a level (ghost-carrying) vector: its ghosts are
// refreshed here; y's ghost plane is compress-added into the owner (CG).
// timed: the launch is bracketed by profiling events (fem_options.profile; only the
// PCG operator apply of cg_solve and the eager fem_apply calls are, so that the
// events do not perturb the timed solve: the kernel is the same in every apply).
// Distributed level: the halo exchanges run on the handle's communication stream and
// overlap the cells that do not touch ghosts (z-slab interior), SURVEY §8e:
//   CG:   zero y | import x ghost plane || cells [0, mid) | wait, top layer |
//         export y ghost plane || cells [mid, top) | wait, add the received plane
//   SIPG: import both ghost layers || interior layers | wait, bottom and top layers
void apply_level_overlap(fem_ctx* h, const Level& L, const double* x, double* y) {
  const int64_t layer = (int64_t)L.n[0] * L.n[1];
  const int n2 = L.n[2];
  cudaStream_t cs = h->comm_stream;
  FEM_CUDA_TRY(cudaEventRecord(h->ev_fork, h->stream));
  FEM_CUDA_TRY(cudaStreamWaitEvent(cs, h->ev_fork, 0));
  halo_import_on(h, L, const_cast<double*>(x), cs);
  FEM_CUDA_TRY(cudaEventRecord(h->ev_import, cs));
  if (is_cg(h)) {
    const int mid = (n2 - 1) / 2;
    launch_cg_apply(h, L, x, y, 0, mid * layer);
    FEM_CUDA_TRY(cudaStreamWaitEvent(h->stream, h->ev_import, 0));
    launch_cg_apply(h, L, x, y, (int64_t)(n2 - 1) * layer, (int64_t)n2 * layer);
    FEM_CUDA_TRY(cudaEventRecord(h->ev_fork, h->stream));
    FEM_CUDA_TRY(cudaStreamWaitEvent(cs, h->ev_fork, 0));
    halo_export_send(h, L, y, cs);
    FEM_CUDA_TRY(cudaEventRecord(h->ev_export, cs));
    launch_cg_apply(h, L, x, y, (int64_t)mid * layer, (int64_t)(n2 - 1) * layer);
    FEM_CUDA_TRY(cudaStreamWaitEvent(h->stream, h->ev_export, 0));
    if (L.ghost_lo >= 0) launch_add(h, y, L.halo, (int64_t)L.nn[0] * L.nn[1]);
  } else {
    if (n2 >= 3) launch_dg_apply(h, L, x, y, layer, (int64_t)(n2 - 1) * layer);
    FEM_CUDA_TRY(cudaStreamWaitEvent(h->stream, h->ev_import, 0));
    launch_dg_apply(h, L, x, y, 0, layer);
    if (n2 >= 2) launch_dg_apply(h, L, x, y, (int64_t)(n2 - 1) * layer, (int64_t)n2 * layer);
  }
}

void apply_level(fem_ctx* h, const Level& L, const double* x, double* y, bool set_constrained = true,
                 bool timed = false) {
  const bool finest = timed && h->prof.mode == 1 && (&L == &h->levels.back());
  if (h->prof.on && finest && !h->prof.capturing && h->prof.used + 2 > 4096) prof_collect(h);
  if (L.dist && h->comm && h->overlap) {
    if (is_cg(h)) {
      if (!(y == L.t && L.t_zero)) launch_zero(h, y, L.n_store);
      if (y == L.t) L.t_zero = false;
      h->y_is_zero = true;
    }
    prof_begin(h, finest);
    apply_level_overlap(h, L, x, y);
    prof_end(h, finest);
    h->y_is_zero = false;
    if (is_cg(h) && set_constrained) launch_set_constrained(h, L, x, y);
    return;
  }
  halo_import(h, L, const_cast<double*>(x));
  if (use_stencil2(h, L)) {   // writes every output once, constrained rows included
    if (y == L.t) L.t_zero = false;
    prof_begin(h, finest);
    launch_cg_stencil_apply(h, L, x, y, set_constrained);
    prof_end(h, finest);
    return;
  }
  if (is_cg(h)) {
    // the Cartesian fast path zeroes y itself, chunk by chunk (kernels_cg.cu)
    const bool tiled = L.cartesian && !h->general_path;
    const bool y_zero = y == L.t && L.t_zero;
    if (!tiled && !y_zero) launch_zero(h, y, L.n_store);
    if (y == L.t) L.t_zero = false;
    h->y_is_zero = y_zero;   // the Cartesian element path zeroes y itself unless told it is zero
    prof_begin(h, finest);
    launch_cg_apply(h, L, x, y);
    h->y_is_zero = false;
    prof_end(h, finest);
    halo_export_add(h, L, y);
    if (set_constrained) launch_set_constrained(h, L, x, y);
  } else {
    prof_begin(h, finest);
    launch_dg_apply(h, L, x, y);
    prof_end(h, finest);
  }
}

// ---------------------------------------------------------------- level transfer
// xc = P^T (bf - axf) from level l to l-1 (axf may be null).  Distributed fine and
// replicated coarse level: the fine residual is gathered (all-reduce of the
// zero-padded owned slices) and restricted on the whole-level twin.
void restrict_to(fem_ctx* h, int l, const double* bf, const double* axf, double* xc) {
  Level& F = h->levels[l];
  Level& C = h->levels[l - 1];
  if (F.dist && !C.dist) {
    launch_zero(h, F.gb, F.n_global);
    launch_sub(h, F.gb + F.first_global, bf, axf, F.n_dofs);
    allreduce(h, F.gb, F.n_global);
    launch_restrict(h, C, *F.full, F.gb, nullptr, xc);
    return;
  }
  launch_restrict(h, C, F, bf, axf, xc);
  halo_export_add(h, C, xc);
}

// xf += P xc from level l-1 to l.  xc must be a level vector of l-1 (ghosts refreshed).
void prolongate_from(fem_ctx* h, int l, double* xc, double* xf) {
  Level& F = h->levels[l];
  Level& C = h->levels[l - 1];
  if (F.dist && !C.dist) {
    launch_zero(h, F.gx, F.n_global);
    launch_prolongate_add(h, C, *F.full, xc, F.gx);
    launch_add(h, xf, F.gx + F.first_global, F.n_dofs);
    return;
  }
  if (is_cg(h)) halo_import(h, C, xc);
  launch_prolongate_add(h, C, F, xc, xf);
}

// ---------------------------------------------------------------- Chebyshev
// x_out = S(x_in, b) on level l (x_in == nullptr: zero start), reading R9/O5:
// x_1 = x_0 + D^-1 (b - A x_0) / theta;  x_{i+1} = x_i + rho_i rho_{i-1} (x_i - x_{i-1})
//        + (2 rho_i / delta) D^-1 (b - A x_i),  rho_i = 1/(2 sigma - rho_{i-1}), rho_0 = 1/sigma.
// Work buffers w[0..2] must differ from x_in/x_out/b.
// CG levels with the fused line kernel (single rank, deformed, default G layout)
// Only small levels: there a smoothing step is latency-bound and one launch instead of
// two saves ~2.5 us; on large levels the wider gather (five streams, 79 registers) costs
// more than the separate elementwise pass (C2 finest: 90 us fused vs 62 + 17 us).
bool cg_fused_ok(const fem_ctx* h, const Level& L) {
  return is_cg(h) && h->fuse_cheb && L.tf[0] && !L.dist && !L.cartesian &&
         (L.glayout == kGLayoutCell || L.glayout == kGLayoutCell8) &&
         L.n_cells <= h->fuse_max_cells;
}

// Chebyshev smoothing with every step but (optionally) the last fused into the CG line
// kernel's gather: kernel j materialises x_j from (x_{j-1}, x_{j-2}, A x_{j-1}) and
// accumulates A x_j into tf[k], clearing tf[k+1] for kernel j+1 (tf[k-1], which kernel j
// read, is free again).  want_ax: the last step is fused too and the buffer holding
// A x_out is returned (the V-cycle's residual); else the last step is the elementwise
// kernel and nullptr is returned.  Arithmetic identical to the unfused recurrence.
double* chebyshev_cg_fused(fem_ctx* h, Level& L, const double* b, const double* x_in, double* x_out,
                           double* w0, double* w1, double* w2, bool want_ax) {
  const int p = h->opt.cheb_degree;
  const double a = h->opt.cheb_hi * L.lam, c = h->opt.cheb_lo * L.lam;
  const double theta = 0.5 * (a + c), delta = 0.5 * (a - c);
  const double sigma = theta / delta;
  double rho = 1.0 / sigma;
  double* bufs[3] = {w0, w1, w2};
  int nb = 0;
  auto next = [&](const double* avoid1, const double* avoid2) {
    for (int i = 0; i < 3; ++i) {
      double* cand = bufs[(nb + i) % 3];
      if (cand != avoid1 && cand != avoid2) {
        nb = (nb + i + 1) % 3;
        return cand;
      }
    }
    return (double*)nullptr;
  };
  int k = 0;
  launch_zero(h, L.tf[0], L.n_store);
  // one fused launch: input x (materialised from it when mat), accumulate into tf[k]
  auto fused = [&](const double* x, const double* xo, double* xnew, double c1, double c2, int mat) {
    CgFuse f;
    f.xo = xo;
    f.b = b;
    f.dinv = L.dinv;
    f.t = L.tf[(k + 2) % 3];
    f.xnew = xnew;
    f.zbuf = L.tf[(k + 1) % 3];
    f.c1 = c1;
    f.c2 = c2;
    f.materialize = mat;
    f.on = 1;
    h->cgf = f;
    launch_cg_apply(h, L, x, L.tf[k]);
    h->cgf = CgFuse{};
    k = (k + 1) % 3;
  };
  const double* x = x_in;
  const double* xo = nullptr;
  if (x_in) fused(x_in, nullptr, nullptr, 0.0, 0.0, 0);   // A x_in
  for (int i = 1; i <= p; ++i) {
    double c1 = 0.0, c2 = 1.0 / theta;
    if (i > 1) {
      const double rho_new = 1.0 / (2.0 * sigma - rho);
      c1 = rho_new * rho;
      c2 = 2.0 * rho_new / delta;
      rho = rho_new;
    }
    double* xn = (i == p) ? x_out : next(x, xo);
    if (i < p || want_ax) {
      fused(x, xo, xn, c1, c2, 1);
    } else {
      // last step, elementwise: A x_{p-1} is in tf[k-1]
      launch_cheb_step(h, L, xn, x, xo, b, x ? L.tf[(k + 2) % 3] : nullptr, c1, c2, xo != nullptr);
    }
    xo = x;
    x = xn;
  }
  return want_ax ? L.tf[(k + 2) % 3] : nullptr;
}

void chebyshev(fem_ctx* h, Level& L, const double* b, const double* x_in, double* x_out,
               double* w0, double* w1, double* w2) {
  if (cg_fused_ok(h, L)) {
    chebyshev_cg_fused(h, L, b, x_in, x_out, w0, w1, w2, false);
    return;
  }
  const int p = h->opt.cheb_degree;
  const double a = h->opt.cheb_hi * L.lam, c = h->opt.cheb_lo * L.lam;
  const double theta = 0.5 * (a + c), delta = 0.5 * (a - c);
  const double sigma = theta / delta;
  double rho = 1.0 / sigma;
  double* bufs[3] = {w0, w1, w2};
  int nb = 0;
  auto next = [&](const double* avoid1, const double* avoid2) {
    for (int i = 0; i < 3; ++i) {
      double* cand = bufs[(nb + i) % 3];
      if (cand != avoid1 && cand != avoid2) {
        nb = (nb + i + 1) % 3;
        return cand;
      }
    }
    return (double*)nullptr;
  };
  const double* xo = nullptr;
  const double* x = nullptr;
  // SIPG: the element-centric apply writes each cell's result once, so the step is fused
  // into its epilogue (no A x vector written and read back, one launch per step)
  // (Cartesian Kronecker kernel only: on the deformed quadrature kernel, which is not
  // memory bound, the four extra epilogue streams cost more than the saved pass, C5 +0.6%)
  const bool fused = !is_cg(h) && h->fuse_cheb && L.cartesian && h->dg_kron;
  const bool st2 = h->fuse_cheb && use_stencil2(h, L);
  // profile mode 2: time every step on the finest level, algorithmic bytes = read x, x_old (if
  // any), b, write x_new (D^-1 from a class table or read: counted as not read)
  const bool tsm = h->prof.mode == 2 && (&L == &h->levels.back());
  auto step = [&](const double* xc, const double* xold, double* xnew, double c1, double c2) {
    if (tsm && !h->prof.capturing && h->prof.used + 2 > 4096) prof_collect(h);
    prof_begin(h, tsm, 8.0 * (double)L.n_dofs * (xold ? 4 : 3));
    if (st2) {   // Chebyshev step in the stencil's epilogue: no A x vector at all
      launch_cg_stencil_cheb(h, L, xc, xold, b, xnew, c1, c2);
    } else if (fused) {
      h->fuse = ChebFuse{xold, b, L.dinv, L.dinv_cls, c1, c2, 1};
      apply_level(h, L, xc, xnew, false);
      h->fuse = ChebFuse{};
    } else {
      apply_level(h, L, xc, L.t, false);
      launch_cheb_step(h, L, xnew, xc, xold, b, L.t, c1, c2, xold != nullptr);
    }
    prof_end(h, tsm);
  };
  // step 1
  double* xn = (p == 1) ? x_out : next(x_in, nullptr);
  if (x_in == nullptr) {
    if (st2 && L.dinv_cls && h->cheb_first_cls)
      launch_cheb_first_cls(h, L, xn, b, 1.0 / theta);
    else
      launch_cheb_step(h, L, xn, nullptr, nullptr, b, nullptr, 0.0, 1.0 / theta, false);
  } else {
    step(x_in, nullptr, xn, 0.0, 1.0 / theta);
  }
  xo = x_in;
  x = xn;
  for (int i = 2; i <= p; ++i) {
    const double rho_new = 1.0 / (2.0 * sigma - rho);
    const double c1 = rho_new * rho, c2 = 2.0 * rho_new / delta;
    rho = rho_new;
    xn = (i == p) ? x_out : next(x, xo);
    step(x, xo, xn, c1, c2);
    xo = x;
    x = xn;
  }
}

void setup_coarse(fem_ctx* h);

// ---------------------------------------------------------------- V-cycle
// x_out = V(l, b).
void vcycle(fem_ctx* h, int l, const double* b, double* x_out) {
  if (l == 0) {
    setup_coarse(h);
    launch_coarse_solve(h, b, x_out);
    return;
  }
  Level& L = h->levels[l];
  Level& C = h->levels[l - 1];
  // pre-smoothing from zero into L.x (x_out may be L.x for coarse levels)
  double* xs = (x_out == L.x) ? L.x2 : L.x;
  double* wa = (x_out == L.x) ? L.x : L.x2;
  // buffers for the smoother: three distinct from b, xs
  // work buffers: x3, b2 and wa (wa may be x_out on coarse levels, which is not live
  // yet; the elementwise Chebyshev update is safe in place)
  // residual, restriction: C.b = P^T (b - A xs)
  if (cg_fused_ok(h, L)) {
    const double* axs = chebyshev_cg_fused(h, L, b, nullptr, xs, L.x3, L.b2, wa, true);
    restrict_to(h, l, b, axs, C.b);
  } else {
    chebyshev(h, L, b, nullptr, xs, L.x3, L.b2, wa);
    apply_level(h, L, xs, L.t, false);
    restrict_to(h, l, b, L.t, C.b);
  }
  vcycle(h, l - 1, C.b, C.x);
  prolongate_from(h, l, C.x, xs);
  chebyshev(h, L, b, xs, x_out, L.x3, L.b2, wa);
}

// ---------------------------------------------------------------- lambda_max
// Largest eigenvalue of a symmetric tridiagonal matrix (bisection, Sturm counts).
double tridiag_max_eig(const std::vector<double>& d, const std::vector<double>& e) {
  const int m = (int)d.size();
  double lo = 1e300, hi = -1e300;
  for (int i = 0; i < m; ++i) {
    double r = (i > 0 ? std::fabs(e[i - 1]) : 0.0) + (i + 1 < m ? std::fabs(e[i]) : 0.0);
    lo = std::min(lo, d[i] - r);
    hi = std::max(hi, d[i] + r);
  }
  auto count_below = [&](double x) {  // number of eigenvalues < x
    int cnt = 0;
    double q = 1.0;
    for (int i = 0; i < m; ++i) {
      q = d[i] - x - (i > 0 ? e[i - 1] * e[i - 1] / q : 0.0);
      if (q == 0.0) q = -1e-300;
      if (q < 0) ++cnt;
    }
    return cnt;
  };
  for (int it = 0; it < 200; ++it) {
    double mid = 0.5 * (lo + hi);
    if (count_below(mid) < m) lo = mid; else hi = mid;
    if (hi - lo <= 1e-15 * std::max(1.0, std::fabs(hi))) break;
  }
  return 0.5 * (lo + hi);
}

// 15 Jacobi-PCG iterations on A s-problem (reading O6).
double estimate_lambda(fem_ctx* h, Level& L) {
  double *s = L.b, *r = L.x, *z = L.x2, *p = L.x3, *q = L.t;
  launch_splitmix(h, L, h->opt.eig_seed, s);
  if (is_cg(h)) launch_set_constrained_value(h, L, 0.0, s);   // Dirichlet entries of s are 0
  launch_copy(h, r, s, L.n_dofs);
  launch_cheb_step(h, L, z, nullptr, nullptr, r, nullptr, 0.0, 1.0, false);  // z = D^-1 r
  launch_copy(h, p, z, L.n_dofs);
  dot(h, L, r, z, 4);
  FEM_CUDA_TRY(cudaMemcpyAsync(h->hscal + 4, h->scal + 4, sizeof(double), cudaMemcpyDeviceToHost, h->stream));
  FEM_CUDA_TRY(cudaStreamSynchronize(h->stream));
  double rz = h->hscal[4];
  std::vector<double> alpha, beta;
  for (int it = 0; it < h->opt.eig_iters; ++it) {
    apply_level(h, L, p, q, false);
    dot(h, L, p, q, 5);
    FEM_CUDA_TRY(cudaMemcpyAsync(h->hscal + 5, h->scal + 5, sizeof(double), cudaMemcpyDeviceToHost, h->stream));
    FEM_CUDA_TRY(cudaStreamSynchronize(h->stream));
    const double pq = h->hscal[5];
    if (!(pq > 0) || !(rz > 0)) break;
    const double a = rz / pq;
    launch_axpby(h, r, q, -a, 1.0, L.n_dofs);                                   // r -= a q
    launch_cheb_step(h, L, z, nullptr, nullptr, r, nullptr, 0.0, 1.0, false);  // z = D^-1 r
    dot(h, L, r, z, 4);
    FEM_CUDA_TRY(cudaMemcpyAsync(h->hscal + 4, h->scal + 4, sizeof(double), cudaMemcpyDeviceToHost, h->stream));
    FEM_CUDA_TRY(cudaStreamSynchronize(h->stream));
    const double rz_new = h->hscal[4];
    alpha.push_back(a);
    beta.push_back(rz_new / rz);
    rz = rz_new;
    if (rz_new == 0.0) break;
    launch_axpby(h, p, z, 1.0, beta.back(), L.n_dofs);                          // p = z + b p
  }
  const int m = (int)alpha.size();
  if (m == 0) throw Error{FEM_E_BREAKDOWN, "Lanczos breakdown on level " + std::to_string(L.idx)};
  std::vector<double> d(m), e(std::max(m - 1, 0));
  for (int j = 0; j < m; ++j) {
    d[j] = 1.0 / alpha[j] + (j > 0 ? beta[j - 1] / alpha[j - 1] : 0.0);
    if (j + 1 < m) e[j] = std::sqrt(beta[j]) / alpha[j];
  }
  double lam = tridiag_max_eig(d, e);
  if (h->comm && !L.dist) {
    // replicated level: every rank ran the same iteration up to rounding (atomics);
    // agree on one value so that all ranks smooth with the same polynomial
    h->hscal[7] = lam;
    FEM_CUDA_TRY(cudaMemcpyAsync(h->scal + 7, h->hscal + 7, sizeof(double), cudaMemcpyHostToDevice, h->stream));
    allreduce(h, h->scal + 7, 1);
    FEM_CUDA_TRY(cudaMemcpyAsync(h->hscal + 7, h->scal + 7, sizeof(double), cudaMemcpyDeviceToHost, h->stream));
    FEM_CUDA_TRY(cudaStreamSynchronize(h->stream));
    lam = h->hscal[7] / h->nranks;
  }
  return lam;
}

// ---------------------------------------------------------------- coarse solve
constexpr int kMaxCoarseFree = 4096;

void setup_coarse(fem_ctx* h) {
  if (h->coarse_inv) return;
  Level& L0 = h->levels[0];
  const int64_t n = L0.n_dofs;
  std::vector<double> diag(n);
  FEM_CUDA_TRY(cudaMemcpyAsync(diag.data(), L0.diag, sizeof(double) * n, cudaMemcpyDeviceToHost, h->stream));
  // free DoFs: CG rows whose dinv is nonzero; all DG DoFs
  std::vector<double> dinv(n);
  FEM_CUDA_TRY(cudaMemcpyAsync(dinv.data(), L0.dinv, sizeof(double) * n, cudaMemcpyDeviceToHost, h->stream));
  FEM_CUDA_TRY(cudaStreamSynchronize(h->stream));
  std::vector<int> fr;
  for (int64_t i = 0; i < n; ++i)
    if (dinv[i] != 0.0) fr.push_back((int)i);
  const int nf = (int)fr.size();
  if (nf > kMaxCoarseFree)
    throw Error{FEM_E_ARG, "coarsest level has " + std::to_string(nf) +
                               " free DoFs (limit " + std::to_string(kMaxCoarseFree) +
                               "); use cell counts divisible by a power of two"};
  std::vector<double> A((size_t)nf * nf), col(n), e(n, 0.0);
  double *de = L0.x, *dy = L0.t;
  for (int j = 0; j < nf; ++j) {
    launch_zero(h, de, n);
    const double one = 1.0;
    FEM_CUDA_TRY(cudaMemcpyAsync(de + fr[j], &one, sizeof(double), cudaMemcpyHostToDevice, h->stream));
    apply_level(h, L0, de, dy, false);
    FEM_CUDA_TRY(cudaMemcpyAsync(col.data(), dy, sizeof(double) * n, cudaMemcpyDeviceToHost, h->stream));
    FEM_CUDA_TRY(cudaStreamSynchronize(h->stream));
    for (int i = 0; i < nf; ++i) A[(size_t)i * nf + j] = col[fr[i]];
  }
  // symmetrise (rounding) and Cholesky A = L L^T
  for (int i = 0; i < nf; ++i)
    for (int j = 0; j < i; ++j) A[(size_t)i * nf + j] = A[(size_t)j * nf + i] =
        0.5 * (A[(size_t)i * nf + j] + A[(size_t)j * nf + i]);
  std::vector<double> Lc((size_t)nf * nf, 0.0);
  for (int j = 0; j < nf; ++j) {
    double s = A[(size_t)j * nf + j];
    for (int k = 0; k < j; ++k) s -= Lc[(size_t)j * nf + k] * Lc[(size_t)j * nf + k];
    if (!(s > 0)) throw Error{FEM_E_BREAKDOWN, "coarse matrix not positive definite"};
    Lc[(size_t)j * nf + j] = std::sqrt(s);
    for (int i = j + 1; i < nf; ++i) {
      double t = A[(size_t)i * nf + j];
      for (int k = 0; k < j; ++k) t -= Lc[(size_t)i * nf + k] * Lc[(size_t)j * nf + k];
      Lc[(size_t)i * nf + j] = t / Lc[(size_t)j * nf + j];
    }
  }
  // A^-1 columns by forward/backward substitution
  std::vector<double> inv((size_t)nf * nf), y(nf);
  for (int c = 0; c < nf; ++c) {
    for (int i = 0; i < nf; ++i) {
      double s = (i == c) ? 1.0 : 0.0;
      for (int k = 0; k < i; ++k) s -= Lc[(size_t)i * nf + k] * y[k];
      y[i] = s / Lc[(size_t)i * nf + i];
    }
    for (int i = nf - 1; i >= 0; --i) {
      double s = y[i];
      for (int k = i + 1; k < nf; ++k) s -= Lc[(size_t)k * nf + i] * inv[(size_t)k * nf + c];
      inv[(size_t)i * nf + c] = s / Lc[(size_t)i * nf + i];
    }
  }
  h->n_coarse_free = nf;
  FEM_CUDA_TRY(cudaMalloc(&h->coarse_free, sizeof(int) * std::max(nf, 1)));
  h->coarse_inv = dalloc((int64_t)nf * nf);
  FEM_CUDA_TRY(cudaMemcpy(h->coarse_free, fr.data(), sizeof(int) * nf, cudaMemcpyHostToDevice));
  std::vector<int> pos(n, -1);
  for (int i = 0; i < nf; ++i) pos[fr[i]] = i;
  FEM_CUDA_TRY(cudaMalloc(&h->coarse_pos, sizeof(int) * std::max<int64_t>(n, 1)));
  FEM_CUDA_TRY(cudaMemcpy(h->coarse_pos, pos.data(), sizeof(int) * n, cudaMemcpyHostToDevice));
  FEM_CUDA_TRY(cudaMemcpy(h->coarse_inv, inv.data(), sizeof(double) * nf * nf, cudaMemcpyHostToDevice));
  // pageable H2D copies may return before the DMA lands, and they are not ordered with
  // a non-blocking h->stream: complete them before coarse_solve_kernel can read them
  FEM_CUDA_TRY(cudaDeviceSynchronize());
}

// ---------------------------------------------------------------- CUDA graphs
struct Captured {
  cudaGraphExec_t exec = nullptr;
  int64_t kernels = 0;
};

template <typename F>
Captured capture(fem_ctx* h, std::vector<std::pair<cudaEvent_t, cudaEvent_t>>& ev, std::vector<double>& evb,
                  F&& body) {
  cudaStream_t user = h->stream;
  Captured c;
  h->stream = h->cap_stream;
  h->prof.capturing = true;
  h->prof.cap = &ev;
  h->prof.capb = &evb;
  g_capture_count = &c.kernels;
  auto restore = [&] {
    h->stream = user;
    h->prof.capturing = false;
    h->prof.cap = nullptr;
    h->prof.capb = nullptr;
    g_capture_count = nullptr;
  };
  // the graph must not rely on buffer state observed at capture time
  for (auto& L : h->levels) L.t_zero = false;
  cudaGraph_t g = nullptr;
  cudaError_t e = cudaStreamBeginCapture(h->cap_stream, cudaStreamCaptureModeThreadLocal);
  if (e != cudaSuccess) {
    restore();
    throw Error{FEM_E_CUDA, std::string("cudaStreamBeginCapture: ") + cudaGetErrorString(e)};
  }
  try {
    body();
  } catch (...) {
    cudaStreamEndCapture(h->cap_stream, &g);
    if (g) cudaGraphDestroy(g);
    restore();
    throw;
  }
  e = cudaStreamEndCapture(h->cap_stream, &g);
  restore();
  if (e != cudaSuccess) throw Error{FEM_E_CUDA, std::string("cudaStreamEndCapture: ") + cudaGetErrorString(e)};
  e = cudaGraphInstantiate(&c.exec, g, 0);
  cudaGraphDestroy(g);
  if (e != cudaSuccess) throw Error{FEM_E_CUDA, std::string("cudaGraphInstantiate: ") + cudaGetErrorString(e)};
  return c;
}

void launch_graph(fem_ctx* h, cudaGraphExec_t g, int64_t kernels) {
  FEM_CUDA_TRY(cudaGraphLaunch(g, h->stream));
  g_launches += kernels;
}

void drop_solve_graphs(fem_ctx* h) {
  if (h->sg.g_pre) cudaGraphExecDestroy(h->sg.g_pre);
  if (h->sg.g_upd) cudaGraphExecDestroy(h->sg.g_upd);
  for (auto* v : {&h->sg.ev_pre, &h->sg.ev_upd}) {
    for (auto& p : *v) {
      cudaEventDestroy(p.first);
      cudaEventDestroy(p.second);
    }
    v->clear();
  }
  h->sg.evb_pre.clear();
  h->sg.evb_upd.clear();
  if (h->sg.g_loop) cudaGraphExecDestroy(h->sg.g_loop);
  h->sg.g_loop = nullptr;
  h->sg.g_pre = h->sg.g_upd = nullptr;
  h->sg.b = nullptr;
  h->sg.x = nullptr;
}

// ---------------------------------------------------------------- setup
// Level hierarchy and z-slab partition (include/fem.h fem_partition): halve while
// every n_d is even and max n_d > coarse_cells; a level is distributed while
// n_z % P == 0 and every rank keeps >= slab_min_layers layers and slab_min_dofs DoFs (the finest level
// always is, for P > 1), coarser levels are replicated.
std::vector<fem_level_part> partition(const fem_mesh& m, int k, int method, const fem_options& o) {
  const int P = m.nranks, r = m.rank;
  if (P < 1 || r < 0 || r >= P) throw Error{FEM_E_ARG, "rank must be in [0, nranks)"};
  if (m.n[2] % P != 0) throw Error{FEM_E_ARG, "n[2] must be divisible by nranks (z-slabs)"};
  std::vector<std::array<int, 3>> ns;
  std::array<int, 3> n = {m.n[0], m.n[1], m.n[2]};
  ns.push_back(n);
  while (n[0] % 2 == 0 && n[1] % 2 == 0 && n[2] % 2 == 0 && std::max(n[0], std::max(n[1], n[2])) > o.coarse_cells) {
    n = {n[0] / 2, n[1] / 2, n[2] / 2};
    ns.push_back(n);
  }
  const int nl = (int)ns.size();
  if (P > 1 && nl < 2)
    throw Error{FEM_E_ARG, "multi-rank needs a mesh that coarsens at least once (the coarsest level is "
                           "replicated on every rank)"};
  std::vector<fem_level_part> out(nl);
  const int64_t N3 = (int64_t)(k + 1) * (k + 1) * (k + 1);
  bool dist = P > 1;
  for (int i = 0; i < nl; ++i) {            // i = 0: finest
    const auto& c = ns[i];
    fem_level_part& q = out[nl - 1 - i];
    if (i > 0) {
      const int64_t lvl_dofs = method == FEM_CG
                                   ? (int64_t)(k * c[0] + 1) * (k * c[1] + 1) * (k * c[2] + 1)
                                   : (int64_t)c[0] * c[1] * c[2] * N3;
      dist = dist && c[2] % P == 0 && c[2] / P >= std::max(1, o.slab_min_layers) &&
             lvl_dofs / P >= o.slab_min_dofs && i < nl - 1;
    }
    const int nzl = dist ? c[2] / P : c[2];
    const int cz0 = dist ? r * nzl : 0;
    for (int d = 0; d < 3; ++d) {
      q.cells[d] = d == 2 ? nzl : c[d];
      q.global_cells[d] = c[d];
    }
    q.cell_z0 = cz0;
    q.distributed = dist ? 1 : 0;
    q.ghost_lo = dist && r > 0 ? r - 1 : -1;
    q.ghost_hi = dist && r < P - 1 ? r + 1 : -1;
    if (method == FEM_CG) {
      const int64_t plane = (int64_t)(k * c[0] + 1) * (k * c[1] + 1);
      q.n_global = plane * (k * c[2] + 1);
      const int64_t own_planes = (int64_t)k * nzl + ((!dist || r == P - 1) ? 1 : 0);
      q.n_owned = own_planes * plane;
      q.first_global = (int64_t)k * cz0 * plane;
      q.n_stored = ((int64_t)k * nzl + 1) * plane;
    } else {
      const int64_t layer = (int64_t)c[0] * c[1] * N3;
      q.n_global = layer * c[2];
      q.n_owned = layer * nzl;
      q.first_global = layer * cz0;
      q.n_stored = q.n_owned + (dist ? 2 * layer : 0);
    }
  }
  return out;
}

void fill_level(fem_ctx* h, Level& L, const fem_level_part& q, int idx) {
  L.idx = idx;
  double det = 1.0;
  for (int d = 0; d < 3; ++d) {
    L.n[d] = q.cells[d];
    L.nn[d] = h->k * q.cells[d] + 1;
    L.h[d] = (h->mesh.hi[d] - h->mesh.lo[d]) / q.global_cells[d];
    det *= 0.5 * L.h[d];
  }
  for (int d = 0; d < 3; ++d) L.cart[d] = det * (2.0 / L.h[d]) * (2.0 / L.h[d]);
  L.nzg = q.global_cells[2];
  L.cz0 = q.cell_z0;
  L.dist = q.distributed != 0;
  L.ghost_lo = q.ghost_lo;
  L.ghost_hi = q.ghost_hi;
  L.n_cells = (int64_t)q.cells[0] * q.cells[1] * q.cells[2];
  L.n_dofs = q.n_owned;
  L.n_store = q.n_stored;
  L.own_off = (!is_cg(h) && L.dist) ? (int64_t)q.cells[0] * q.cells[1] * (h->k + 1) * (h->k + 1) * (h->k + 1) : 0;
  L.first_global = q.first_global;
  L.n_global = q.n_global;
  L.cartesian = (h->mesh.deform_eps == 0.0) && !mesh_general(h->mesh);
}

void build_levels(fem_ctx* h) {
  const std::vector<fem_level_part> parts = partition(h->mesh, h->k, h->method, h->opt);
  const int nl = (int)parts.size();
  h->levels.resize(nl);
  for (int l = 0; l < nl; ++l) {
    Level& L = h->levels[l];
    fill_level(h, L, parts[l], l);
    L.diag = valloc(L);
    L.dinv = valloc(L);
    L.b = valloc(L);
    L.x = valloc(L);
    L.t = valloc(L);
    L.x2 = valloc(L);
    L.x3 = valloc(L);
    L.b2 = valloc(L);
    if (is_cg(h) && h->fuse_cheb && !L.dist && !L.cartesian && L.n_cells <= h->fuse_max_cells)
      for (double*& t : L.tf) t = valloc(L);
    if (L.dist && is_cg(h)) L.halo = dalloc((int64_t)L.nn[0] * L.nn[1]);
    if (L.dist && l > 0 && !parts[l - 1].distributed) {
      // last distributed level: whole-level twin for the transfers to the replicated level
      fem_level_part whole = parts[l];
      whole.cells[2] = whole.global_cells[2];
      whole.cell_z0 = 0;
      whole.distributed = 0;
      whole.ghost_lo = whole.ghost_hi = -1;
      whole.n_owned = whole.n_stored = whole.n_global;
      whole.first_global = 0;
      L.full.reset(new Level());
      fill_level(h, *L.full, whole, l);
      L.gb = dalloc(L.n_global);
      L.gx = dalloc(L.n_global);
    }
  }
}

void level_geometry_and_diagonal(fem_ctx* h, Level& L) {
  const int N = h->k + 1;
  if (!L.cartesian) {
    L.glayout = !is_cg(h) ? kGLayoutCell
                : (h->k <= 4 && h->plane_kernel) ? kGLayoutPlane
                : h->dbasis ? kGLayoutXLine
                : (h->k == 4 && h->line_cell_fast) ? kGLayoutCell8 : kGLayoutCell;
    const bool plane = L.glayout == kGLayoutPlane, c8 = L.glayout == kGLayoutCell8;
    const int64_t cells = plane ? (L.n_cells + kGroupCells - 1) / kGroupCells * kGroupCells
                          : c8 ? (L.n_cells + kCell8 - 1) / kCell8 * kCell8 : L.n_cells;
    L.G = dalloc(cells * 6 * N * N * N);
    if (plane || c8) {
      FEM_CUDA_TRY(cudaMemset(L.G, 0, sizeof(double) * cells * 6 * N * N * N));
      FEM_CUDA_TRY(cudaDeviceSynchronize());   // legacy-stream memset vs launch_geometry on h->stream
    }
    const unsigned long long init = std::numeric_limits<unsigned long long>::max();
    FEM_CUDA_TRY(cudaMemcpyAsync(h->geom_err, &init, sizeof(init), cudaMemcpyHostToDevice, h->stream));
    launch_geometry(h, L);
    unsigned long long bad = 0;
    FEM_CUDA_TRY(cudaMemcpyAsync(&bad, h->geom_err, sizeof(bad), cudaMemcpyDeviceToHost, h->stream));
    FEM_CUDA_TRY(cudaStreamSynchronize(h->stream));
    if (bad != init)
      throw Error{FEM_E_GEOMETRY, "det J <= 0 on level " + std::to_string(L.idx) + " in cell " +
                                      std::to_string(bad)};
    if (!is_cg(h)) launch_dg_face_geometry(h, L);
  }
  if (is_cg(h)) {
    launch_zero(h, L.diag, L.n_store);
    launch_cg_diagonal(h, L);
    halo_export_add(h, L, L.diag);
    launch_set_constrained(h, L, nullptr, L.diag);     // diag = 1 on constrained rows
    launch_dinv(h, L);
    launch_set_constrained_value(h, L, 0.0, L.dinv);   // D^-1 = 0 on constrained rows
    if (use_stencil2(h, L)) {
      // Cartesian CG: D^-1 depends on a node only through its class per direction,
      // 0 (first node), r = 1..k-1 (inside an element), k (interior vertex), k+1 (last
      // node); the fused stencil epilogue reads it from this (k+2)^3 table, copied from
      // the computed D^-1 at one representative node per class
      const int K = h->k, nc = K + 2;
      L.dinv_cls = dalloc((int64_t)nc * nc * nc);
      auto rep = [&](int d, int cl) {
        if (cl == 0) return 0;
        if (cl == K + 1) return L.nn[d] - 1;
        return (cl == K && L.n[d] < 2) ? 0 : cl;
      };
      for (int c2 = 0; c2 < nc; ++c2)
        for (int c1 = 0; c1 < nc; ++c1)
          for (int c0 = 0; c0 < nc; ++c0) {
            const int64_t node = rep(0, c0) + (int64_t)L.nn[0] * (rep(1, c1) + (int64_t)L.nn[1] * rep(2, c2));
            FEM_CUDA_TRY(cudaMemcpyAsync(L.dinv_cls + c0 + nc * (c1 + nc * c2), L.dinv + node, sizeof(double),
                                         cudaMemcpyDeviceToDevice, h->stream));
          }
    }
  } else {
    launch_dg_diagonal(h, L);
    launch_dinv(h, L);
    if (L.cartesian && !L.dist && h->dinv_classes) {
      // class c_d = 0 (first cell along d), 1 (interior), 2 (last); representative cells
      const int64_t n3 = (int64_t)(h->k + 1) * (h->k + 1) * (h->k + 1);
      L.dinv_cls = dalloc(27 * n3);
      for (int c2 = 0; c2 < 3; ++c2)
        for (int c1 = 0; c1 < 3; ++c1)
          for (int c0 = 0; c0 < 3; ++c0) {
            const int cc[3] = {c0, c1, c2};
            int rep[3];
            for (int d = 0; d < 3; ++d)
              rep[d] = cc[d] == 0 ? 0 : (cc[d] == 2 ? L.n[d] - 1 : (L.n[d] >= 3 ? 1 : 0));
            const int64_t cell = rep[0] + (int64_t)L.n[0] * (rep[1] + (int64_t)L.n[1] * rep[2]);
            FEM_CUDA_TRY(cudaMemcpyAsync(L.dinv_cls + (c0 + 3 * c1 + 9 * c2) * n3, L.dinv + cell * n3,
                                         sizeof(double) * n3, cudaMemcpyDeviceToDevice, h->stream));
          }
    }
  }
}

struct Staged {
  fem_ctx* h;
  double* dev;
  const double* host_in;
  double* host_out;
  int64_t n;
};

bool is_device_ptr(const void* p) {
  cudaPointerAttributes at;
  cudaError_t e = cudaPointerGetAttributes(&at, p);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

void ensure_stage(fem_ctx* h, int64_t n) {
  if (h->stage_len >= n) return;
  for (auto& s : h->stage) dfree(s);
  for (auto& s : h->stage) s = dalloc(n);
  h->stage_len = n;
}

// Resolve a caller vector to a device pointer (copy-in for host inputs).
const double* in_vec(fem_ctx* h, const double* p, int64_t n, int slot) {
  if (is_device_ptr(p)) return p;
  ensure_stage(h, n);
  FEM_CUDA_TRY(cudaMemcpyAsync(h->stage[slot], p, sizeof(double) * n, cudaMemcpyHostToDevice, h->stream));
  return h->stage[slot];
}

double* out_vec(fem_ctx* h, double* p, int64_t n, int slot, bool copy_in, bool* staged) {
  if (is_device_ptr(p)) {
    *staged = false;
    return p;
  }
  ensure_stage(h, n);
  *staged = true;
  if (copy_in)
    FEM_CUDA_TRY(cudaMemcpyAsync(h->stage[slot], p, sizeof(double) * n, cudaMemcpyHostToDevice, h->stream));
  return h->stage[slot];
}

void finish_out(fem_ctx* h, double* host, const double* dev, int64_t n, bool staged) {
  if (!staged) return;
  FEM_CUDA_TRY(cudaMemcpyAsync(host, dev, sizeof(double) * n, cudaMemcpyDeviceToHost, h->stream));
  FEM_CUDA_TRY(cudaStreamSynchronize(h->stream));
}

void check_handle(fem_handle h) {
  if (!h) throw Error{FEM_E_ARG, "null handle"};
  FEM_CUDA_TRY(cudaSetDevice(h->device));
}

void check_size(int64_t got, int64_t want, const char* what) {
  if (got != want)
    throw Error{FEM_E_SIZE, std::string(what) + ": length " + std::to_string(got) + ", expected " +
                                std::to_string(want)};
}

Level& level_at(fem_handle h, int32_t level) {
  if (level < 0 || level >= (int)h->levels.size())
    throw Error{FEM_E_ARG, "level " + std::to_string(level) + " out of range"};
  return h->levels[level];
}

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return FEM_OK;
  } catch (const Error& e) {
    set_error(e.msg);
    return e.code;
  } catch (const std::bad_alloc&) {
    set_error("host allocation failed");
    return FEM_E_OOM;
  } catch (const std::exception& e) {
    set_error(e.what());
    return FEM_E_ARG;
  }
}

void destroy(fem_ctx* h) {
  if (!h) return;
  cudaSetDevice(h->device);
  if (h->stream) cudaStreamSynchronize(h->stream);
  for (auto& L : h->levels) {
    for (double** p : {&L.G, &L.face, &L.halo, &L.gb, &L.gx, &L.dinv_cls}) dfree(*p);
    for (double** p : {&L.diag, &L.dinv, &L.b, &L.x, &L.x2, &L.x3, &L.t, &L.b2, &L.pcg_r, &L.pcg_p,
                       &L.pcg_q, &L.pcg_z, &L.tf[0], &L.tf[1], &L.tf[2]})
      vfree(L, *p);
  }
  h->comm.reset();
  for (cudaEvent_t e : {h->ev_fork, h->ev_import, h->ev_export})
    if (e) cudaEventDestroy(e);
  if (h->comm_stream) cudaStreamDestroy(h->comm_stream);
  if (h->coarse_free) cudaFree(h->coarse_free);
  if (h->coarse_pos) cudaFree(h->coarse_pos);
  dfree(h->coarse_inv);
  dfree(h->red);
  dfree(h->scal);
  dfree(h->sg.hist_dev);
  if (h->hscal) cudaFreeHost(h->hscal);
  for (auto& s : h->stage) dfree(s);
  if (h->geom_err) cudaFree(h->geom_err);
  for (auto e : h->prof.ev) cudaEventDestroy(e);
  drop_solve_graphs(h);
  if (h->cap_stream) cudaStreamDestroy(h->cap_stream);
  delete h;
}

}  // namespace
}  // namespace fem

using namespace fem;

// On-device stopping test of the conditional PCG loop (R11, reading R13): scal[1] = (p, q),
// scal[2] = (r, r) of this iteration, scal[6] = (b, b); scal[8] counts iterations, scal[9] flags a
// breakdown, scal[10] = rtol, scal[11] = maxit; the relative residual goes to hist[it].
__global__ void pcg_cond_kernel(cudaGraphConditionalHandle hc, double* scal, double* hist) {
  const double pq = scal[1], rn = sqrt(scal[2]), bn = sqrt(scal[6]);
  const double it = scal[8] + 1.0;
  scal[8] = it;
  const double rel = bn > 0 ? rn / bn : rn;
  hist[(int)it] = rel;
  scal[12] = rel;
  const bool bad = !(pq > 0) || !isfinite(rn);
  if (bad) scal[9] = 1.0;
  cudaGraphSetConditional(hc, (!bad && rel > scal[10] && it < scal[11]) ? 1u : 0u);
}

namespace fem {
// Build g_loop (see SolveGraphs).  Returns false (and remembers it) if the driver rejects the
// conditional body, so that the host loop runs instead.
template <typename F1, typename F2>
bool build_cond_loop(fem_ctx* h, F1&& body_pre, F2&& body_upd) {
  if (h->sg.cond_failed) return false;
  cudaGraph_t g = nullptr;
  cudaStream_t user = h->stream;
  auto fail = [&](cudaGraph_t gg) {
    if (gg) cudaGraphDestroy(gg);
    cudaGetLastError();
    h->stream = user;
    g_capture_count = nullptr;
    h->sg.cond_failed = true;
    return false;
  };
  if (cudaGraphCreate(&g, 0) != cudaSuccess) return fail(nullptr);
  cudaGraphConditionalHandle hc;
  if (cudaGraphConditionalHandleCreate(&hc, g, 1, cudaGraphCondAssignDefault) != cudaSuccess) return fail(g);
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = hc;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t node;
  if (cudaGraphAddNode(&node, g, nullptr, 0, &cp) != cudaSuccess) return fail(g);
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  if (!h->sg.hist_dev) h->sg.hist_dev = dalloc(kCondHist);
  int64_t kernels = 0;
  g_capture_count = &kernels;
  h->stream = h->cap_stream;
  for (auto& L : h->levels) L.t_zero = false;
  if (cudaStreamBeginCaptureToGraph(h->cap_stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal) !=
      cudaSuccess)
    return fail(g);
  bool ok = true;
  try {
    body_pre();
    body_upd();
    pcg_cond_kernel<<<1, 1, 0, h->cap_stream>>>(hc, h->scal, h->sg.hist_dev);
    ++kernels;
  } catch (...) {
    ok = false;
  }
  cudaGraph_t out = body;
  const cudaError_t e = cudaStreamEndCapture(h->cap_stream, &out);
  h->stream = user;
  g_capture_count = nullptr;
  if (!ok || e != cudaSuccess) return fail(g);
  if (cudaGraphInstantiate(&h->sg.g_loop, g, 0) != cudaSuccess) {
    h->sg.g_loop = nullptr;
    return fail(g);
  }
  cudaGraphDestroy(g);
  h->sg.k_iter = kernels;
  return true;
}
}  // namespace fem

extern "C" {

const char* fem_last_error(void) { return g_last_error.c_str(); }

int64_t fem_kernel_launches(void) { return g_launches.load(); }

int fem_default_options(fem_options* o) {
  if (!o) {
    set_error("null options");
    return FEM_E_ARG;
  }
  std::memset(o, 0, sizeof(*o));
  o->penalty_factor = 2.0;
  o->cheb_degree = 5;
  o->cheb_lo = 0.06;
  o->cheb_hi = 1.2;
  o->eig_iters = 15;
  o->coarse_cells = 1;
  o->eig_seed = 0x5eed;
  o->lambda_override = nullptr;
  o->stream = nullptr;
  o->device = -1;
  o->profile = 0;
  o->slab_min_layers = 1;
  o->slab_min_dofs = 32768;
  return FEM_OK;
}

int fem_setup(const fem_mesh* mesh, int32_t degree, int32_t method, const fem_options* opt,
              fem_handle* out) {
  fem_ctx* h = nullptr;
  int rc = guarded([&] {
    if (!mesh || !out) throw Error{FEM_E_ARG, "null mesh or output handle"};
    if (degree < 1 || degree > kMaxDeg) throw Error{FEM_E_ARG, "degree must be in [1, 8]"};
    if (method != FEM_CG && method != FEM_SIPG) throw Error{FEM_E_ARG, "method must be FEM_CG or FEM_SIPG"};
    for (int d = 0; d < 3; ++d) {
      if (mesh->n[d] < 1) throw Error{FEM_E_ARG, "cells per direction must be >= 1"};
      if (!(mesh->hi[d] > mesh->lo[d])) throw Error{FEM_E_ARG, "box must have hi > lo"};
    }
    for (int s = 0; s < 6; ++s)
      if (mesh->bc[s] != FEM_BC_DIRICHLET && mesh->bc[s] != FEM_BC_NEUMANN)
        throw Error{FEM_E_ARG, "bc must be FEM_BC_DIRICHLET or FEM_BC_NEUMANN"};
    if (mesh->nranks < 1 || mesh->rank < 0 || mesh->rank >= mesh->nranks)
      throw Error{FEM_E_ARG, "rank must be in [0, nranks)"};
    if (mesh->nranks > 1 && ((mesh->nccl_id != nullptr) == (mesh->local_group != nullptr)))
      throw Error{FEM_E_ARG, "nranks > 1 needs exactly one of nccl_id / local_group"};
    if (mesh->geometry != FEM_GEOM_BOX && mesh->geometry != FEM_GEOM_SHELL)
      throw Error{FEM_E_ARG, "geometry must be FEM_GEOM_BOX or FEM_GEOM_SHELL"};
    if (mesh->mapping_degree < 0 || mesh->mapping_degree > 8)
      throw Error{FEM_E_ARG, "mapping_degree must be in [0, 8]"};
    if (!std::isfinite(mesh->kappa_amplitude)) throw Error{FEM_E_ARG, "kappa_amplitude must be finite"};
    h = new fem_ctx();
    h->k = degree;
    h->method = method;
    h->mesh = *mesh;
    fem_default_options(&h->opt);
    if (opt) h->opt = *opt;
    if (h->opt.cheb_degree < 1 || h->opt.eig_iters < 1 || h->opt.coarse_cells < 1 ||
        !(h->opt.cheb_hi > h->opt.cheb_lo) || !(h->opt.cheb_lo > 0) || !(h->opt.penalty_factor > 0))
      throw Error{FEM_E_ARG, "invalid solver options"};
    if (h->opt.device >= 0) FEM_CUDA_TRY(cudaSetDevice(h->opt.device));
    FEM_CUDA_TRY(cudaGetDevice(&h->device));
    h->stream = (cudaStream_t)h->opt.stream;
    h->rank = mesh->rank;
    h->nranks = mesh->nranks;
    if (h->nranks > 1) {
      h->comm = mesh->nccl_id ? make_nccl_comm(mesh->nccl_id, h->rank, h->nranks)
                              : make_local_comm(mesh->local_group, h->rank, h->nranks);
      h->use_graphs = h->comm->graph_capturable();
      FEM_CUDA_TRY(cudaStreamCreateWithFlags(&h->comm_stream, cudaStreamNonBlocking));
      for (cudaEvent_t* e : {&h->ev_fork, &h->ev_import, &h->ev_export})
        FEM_CUDA_TRY(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    }
    if (const char* e = std::getenv("FEM_OVERLAP")) h->overlap = std::atoi(e) != 0;
    if (const char* e = std::getenv("FEM_NO_GRAPHS")) h->use_graphs = h->use_graphs && std::atoi(e) == 0;
    FEM_CUDA_TRY(cudaStreamCreateWithFlags(&h->cap_stream, cudaStreamNonBlocking));
    h->prof.on = h->opt.profile != 0;
    h->prof.mode = h->opt.profile;
    if (const char* e = std::getenv("FEM_GENERAL_PATH")) h->general_path = std::atoi(e) != 0;
    if (const char* e = std::getenv("FEM_CHUNK_LAYERS")) h->chunk_layers = std::atoi(e);
    if (const char* e = std::getenv("FEM_PLANE")) h->plane_kernel = std::atoi(e) != 0;
    // the block's G chunk staged by one TMA bulk copy beats direct loads at Q4 (8-cell block
    // order: C2 apply 59.4 -> 57.5 us, solve 7.12 -> 6.94 ms) and at k = 7, 8 (deformed
    // apply at ~16M DoFs 692 -> 416 us, 595 -> 498 us); k = 3, 5, 6 are faster direct
    h->g_direct = !((degree == 4 && h->line_cell_fast) || degree == 7 || degree == 8);
    if (const char* e = std::getenv("FEM_G_DIRECT")) h->g_direct = std::atoi(e) != 0;
    if (const char* e = std::getenv("FEM_TMA_MIN_BLOCKS")) h->tma_min_blocks = std::atoll(e);
    if (const char* e = std::getenv("FEM_DBASIS")) h->dbasis = std::atoi(e) != 0;
    if (const char* e = std::getenv("FEM_STENCIL")) h->stencil = std::atoi(e) != 0;
    if (const char* e = std::getenv("FEM_PDL")) h->pdl = std::atoi(e) != 0;
    if (const char* e = std::getenv("FEM_DG_KRON")) h->dg_kron = std::atoi(e) != 0;
    if (const char* e = std::getenv("FEM_FUSE_CHEB")) h->fuse_cheb = std::atoi(e) != 0;
    if (const char* e = std::getenv("FEM_DINV_CLASSES")) h->dinv_classes = std::atoi(e) != 0;
    if (const char* e = std::getenv("FEM_FUSE_CELLS")) h->fuse_max_cells = std::atoll(e);
    if (const char* e = std::getenv("FEM_STENCIL2")) h->stencil2 = std::atoi(e) != 0;
    if (const char* e = std::getenv("FEM_DG_FGEO_FLY")) h->dg_fgeo_fly = std::atoi(e) != 0;
    if (const char* e = std::getenv("FEM_DG_CGEO_FLY")) h->dg_cgeo_fly = std::atoi(e) != 0;
    if (const char* e = std::getenv("FEM_CG_GEO_FLY")) h->cg_geo_fly = std::atoi(e) != 0;
    if (const char* e = std::getenv("FEM_ST_MIN_CELLS")) h->stencil2_min_cells = std::atoll(e);
    if (const char* e = std::getenv("FEM_GT_MIN_CELLS")) h->grid_transfer_min_cells = std::atoll(e);
    if (const char* e = std::getenv("FEM_CHEB_FIRST_CLS")) h->cheb_first_cls = std::atoi(e) != 0;
    if (const char* e = std::getenv("FEM_ST_EZ")) h->stencil_ez = std::atoi(e);
    build_tables(degree, h->tab);
    h->red = dalloc(16 * kRedBlocks + 16);   // partial sums + 16 reduction counters (zeroed)
    FEM_CUDA_TRY(cudaMemset(h->red, 0, sizeof(double) * (16 * kRedBlocks + 16)));
    h->scal = dalloc(16);
    FEM_CUDA_TRY(cudaMemset(h->scal, 0, sizeof(double) * 16));
    FEM_CUDA_TRY(cudaDeviceSynchronize());   // legacy-stream memsets vs kernels on h->stream
    FEM_CUDA_TRY(cudaMallocHost(&h->hscal, sizeof(double) * 16));
    FEM_CUDA_TRY(cudaMalloc(&h->geom_err, sizeof(unsigned long long)));
    build_levels(h);
    for (auto& L : h->levels) level_geometry_and_diagonal(h, L);
    for (size_t l = 1; l < h->levels.size(); ++l) {
      Level& L = h->levels[l];
      L.lam = h->opt.lambda_override ? h->opt.lambda_override[l] : estimate_lambda(h, L);
    }
    FEM_CUDA_TRY(cudaStreamSynchronize(h->stream));
    // (the coarse Cholesky factor is built on first use: setup_coarse)
    // profiling counts only what happens after setup
    h->prof.used = 0;
    h->prof.ms = 0;
    h->prof.launches = 0;
    *out = h;
  });
  if (rc != FEM_OK) destroy(h);
  return rc;
}

int fem_partition(const fem_mesh* mesh, int32_t degree, int32_t method, const fem_options* opt,
                  fem_level_part* out, int32_t max_levels, int32_t* n_levels) {
  return guarded([&] {
    if (!mesh || !out || !n_levels) throw Error{FEM_E_ARG, "null argument"};
    if (degree < 1 || degree > kMaxDeg) throw Error{FEM_E_ARG, "degree must be in [1, 8]"};
    if (method != FEM_CG && method != FEM_SIPG) throw Error{FEM_E_ARG, "method must be FEM_CG or FEM_SIPG"};
    for (int d = 0; d < 3; ++d)
      if (mesh->n[d] < 1) throw Error{FEM_E_ARG, "cells per direction must be >= 1"};
    fem_options o;
    fem_default_options(&o);
    if (opt) o = *opt;
    if (o.coarse_cells < 1) throw Error{FEM_E_ARG, "invalid solver options"};
    const auto parts = partition(*mesh, degree, method, o);
    if ((int)parts.size() > max_levels) throw Error{FEM_E_ARG, "max_levels too small"};
    for (size_t i = 0; i < parts.size(); ++i) out[i] = parts[i];
    *n_levels = (int32_t)parts.size();
  });
}

int fem_info(fem_handle h, int64_t* n_local, int64_t* n_global, int64_t* first_global,
             int32_t* n_levels) {
  return guarded([&] {
    check_handle(h);
    const Level& L = h->levels.back();
    if (n_local) *n_local = L.n_dofs;
    if (n_global) *n_global = L.n_global;
    if (first_global) *first_global = L.first_global;
    if (n_levels) *n_levels = (int32_t)h->levels.size();
  });
}

int fem_level_info(fem_handle h, int32_t level, int64_t* n_dofs, int32_t cells[3]) {
  return guarded([&] {
    check_handle(h);
    const Level& L = level_at(h, level);
    if (n_dofs) *n_dofs = L.n_dofs;
    if (cells)
      for (int d = 0; d < 3; ++d) cells[d] = L.n[d];
  });
}

int fem_level_apply(fem_handle h, int32_t level, const double* x, int64_t nx, double* y, int64_t ny) {
  return guarded([&] {
    check_handle(h);
    Level& L = level_at(h, level);
    if (!x || !y) throw Error{FEM_E_ARG, "null vector"};
    check_size(nx, L.n_dofs, "x");
    check_size(ny, L.n_dofs, "y");
    const double* dx = in_vec(h, x, nx, 0);
    bool st;
    double* dy = out_vec(h, y, ny, 1, false, &st);
    if (L.dist) {   // level vectors carry the ghosts
      launch_copy(h, L.x2, dx, L.n_dofs);
      apply_level(h, L, L.x2, L.t, true, true);
      launch_copy(h, dy, L.t, L.n_dofs);
    } else {
      apply_level(h, L, dx, dy, true, true);
    }
    finish_out(h, y, dy, ny, st);
  });
}

int fem_apply(fem_handle h, const double* x, int64_t nx, double* y, int64_t ny) {
  if (!h) {
    set_error("null handle");
    return FEM_E_ARG;
  }
  return fem_level_apply(h, (int32_t)h->levels.size() - 1, x, nx, y, ny);
}

int fem_level_diagonal(fem_handle h, int32_t level, double* d, int64_t nd) {
  return guarded([&] {
    check_handle(h);
    Level& L = level_at(h, level);
    if (!d) throw Error{FEM_E_ARG, "null vector"};
    check_size(nd, L.n_dofs, "d");
    bool st;
    double* dd = out_vec(h, d, nd, 0, false, &st);
    launch_copy(h, dd, L.diag, L.n_dofs);
    finish_out(h, d, dd, nd, st);
  });
}

int fem_diagonal(fem_handle h, double* d, int64_t nd) {
  if (!h) {
    set_error("null handle");
    return FEM_E_ARG;
  }
  return fem_level_diagonal(h, (int32_t)h->levels.size() - 1, d, nd);
}

int fem_level_lambda(fem_handle h, int32_t level, double* lam) {
  return guarded([&] {
    check_handle(h);
    Level& L = level_at(h, level);
    if (level < 1) throw Error{FEM_E_ARG, "the coarsest level has no smoother"};
    if (!lam) throw Error{FEM_E_ARG, "null output"};
    *lam = L.lam;
  });
}

int fem_level_geometry(fem_handle h, int32_t level, double* G, int64_t nG) {
  return guarded([&] {
    check_handle(h);
    Level& L = level_at(h, level);
    const int N = h->k + 1;
    const int64_t nq = (int64_t)N * N * N;
    check_size(nG, L.n_cells * 6 * nq, "G");
    if (!G) throw Error{FEM_E_ARG, "null vector"};
    if (!L.cartesian && L.glayout == kGLayoutCell) {
      bool st;
      double* dG = out_vec(h, G, nG, 0, false, &st);
      launch_copy(h, dG, L.G, nG);
      finish_out(h, G, dG, nG, st);
      return;
    }
    if (!L.cartesian) {
      // internal layout: permute to the documented [cell][6][q] order on the host
      const int64_t cells = L.glayout == kGLayoutPlane ? (L.n_cells + kGroupCells - 1) / kGroupCells * kGroupCells
                            : L.glayout == kGLayoutCell8 ? (L.n_cells + kCell8 - 1) / kCell8 * kCell8
                                                         : L.n_cells;
      std::vector<double> raw(cells * 6 * nq), out(nG);
      FEM_CUDA_TRY(cudaMemcpyAsync(raw.data(), L.G, sizeof(double) * raw.size(), cudaMemcpyDeviceToHost, h->stream));
      FEM_CUDA_TRY(cudaStreamSynchronize(h->stream));
      for (int64_t c = 0; c < L.n_cells; ++c)
        for (int comp = 0; comp < 6; ++comp)
          for (int q = 0; q < nq; ++q) {
            const int64_t N2 = (int64_t)N * N;
            int64_t src;
            if (L.glayout == kGLayoutXLine) {
              src = (c * 6 + comp) * nq + (q % N) * N2 + q / N;
            } else if (L.glayout == kGLayoutCell8) {
              src = (((c / kCell8) * 6 + comp) * nq + q) * kCell8 + c % kCell8;
            } else {   // plane
              const int64_t g = c / kGroupCells, ci = c % kGroupCells;
              src = (((g * 6 + comp) * N2 + q % N2) * kGroupCells + ci) * N + q / N2;
            }
            out[(c * 6 + comp) * nq + q] = raw[src];
          }
      if (is_device_ptr(G))
      {
        FEM_CUDA_TRY(cudaMemcpy(G, out.data(), sizeof(double) * nG, cudaMemcpyHostToDevice));
        FEM_CUDA_TRY(cudaDeviceSynchronize());
      } else
        std::memcpy(G, out.data(), sizeof(double) * nG);
      return;
    }
    // Cartesian: expand the per-level constants on the host
    std::vector<double> hostG(nG, 0.0);
    for (int64_t c = 0; c < L.n_cells; ++c)
      for (int64_t q = 0; q < nq; ++q) {
        const int q0 = (int)(q % N), q1 = (int)((q / N) % N), q2 = (int)(q / (N * N));
        const double w = h->tab.qw[q0] * h->tab.qw[q1] * h->tab.qw[q2];
        hostG[c * 6 * nq + 0 * nq + q] = L.cart[0] * w;
        hostG[c * 6 * nq + 3 * nq + q] = L.cart[1] * w;
        hostG[c * 6 * nq + 5 * nq + q] = L.cart[2] * w;
      }
    if (is_device_ptr(G))
    {
      FEM_CUDA_TRY(cudaMemcpy(G, hostG.data(), sizeof(double) * nG, cudaMemcpyHostToDevice));
      FEM_CUDA_TRY(cudaDeviceSynchronize());
    } else
      std::memcpy(G, hostG.data(), sizeof(double) * nG);
  });
}

int mg_smooth(fem_handle h, int32_t level, const double* b, int64_t nb, double* x, int64_t nx,
              int32_t x_is_zero) {
  return guarded([&] {
    check_handle(h);
    Level& L = level_at(h, level);
    if (level < 1) throw Error{FEM_E_ARG, "smoothing needs level >= 1"};
    if (!b || !x) throw Error{FEM_E_ARG, "null vector"};
    check_size(nb, L.n_dofs, "b");
    check_size(nx, L.n_dofs, "x");
    const double* db = in_vec(h, b, nb, 0);
    bool st;
    double* dx = out_vec(h, x, nx, 1, !x_is_zero, &st);
    // copy inputs into level buffers so the smoother's work buffers never alias them
    launch_copy(h, L.b, db, L.n_dofs);
    if (!x_is_zero) launch_copy(h, L.x, dx, L.n_dofs);
    chebyshev(h, L, L.b, x_is_zero ? nullptr : L.x, dx, L.x2, L.x3, L.b2);
    finish_out(h, x, dx, nx, st);
  });
}

int mg_prolongate_add(fem_handle h, int32_t level, const double* xc, int64_t nc, double* xf,
                      int64_t nf) {
  return guarded([&] {
    check_handle(h);
    Level& F = level_at(h, level);
    if (level < 1) throw Error{FEM_E_ARG, "prolongation needs level >= 1"};
    Level& C = h->levels[level - 1];
    if (!xc || !xf) throw Error{FEM_E_ARG, "null vector"};
    check_size(nc, C.n_dofs, "xc");
    check_size(nf, F.n_dofs, "xf");
    const double* dc = in_vec(h, xc, nc, 0);
    bool st;
    double* df = out_vec(h, xf, nf, 1, true, &st);
    launch_copy(h, C.x, dc, C.n_dofs);   // level vector: ghosts are imported into it
    prolongate_from(h, level, C.x, df);
    finish_out(h, xf, df, nf, st);
  });
}

int mg_restrict(fem_handle h, int32_t level, const double* xf, int64_t nf, double* xc, int64_t nc) {
  return guarded([&] {
    check_handle(h);
    Level& F = level_at(h, level);
    if (level < 1) throw Error{FEM_E_ARG, "restriction needs level >= 1"};
    Level& C = h->levels[level - 1];
    if (!xc || !xf) throw Error{FEM_E_ARG, "null vector"};
    check_size(nc, C.n_dofs, "xc");
    check_size(nf, F.n_dofs, "xf");
    const double* df = in_vec(h, xf, nf, 0);
    bool st;
    double* dc = out_vec(h, xc, nc, 1, false, &st);
    restrict_to(h, level, df, nullptr, C.b);   // level vector: CG ghost plane compress-added
    launch_copy(h, dc, C.b, C.n_dofs);
    finish_out(h, xc, dc, nc, st);
  });
}

int mg_coarse_solve(fem_handle h, const double* b, int64_t nb, double* x, int64_t nx) {
  return guarded([&] {
    check_handle(h);
    Level& L0 = h->levels[0];
    if (!b || !x) throw Error{FEM_E_ARG, "null vector"};
    check_size(nb, L0.n_dofs, "b");
    check_size(nx, L0.n_dofs, "x");
    setup_coarse(h);
    const double* db = in_vec(h, b, nb, 0);
    bool st;
    double* dx = out_vec(h, x, nx, 1, false, &st);
    launch_coarse_solve(h, db, dx);
    finish_out(h, x, dx, nx, st);
  });
}

int mg_vcycle(fem_handle h, const double* r, int64_t nr, double* z, int64_t nz) {
  return guarded([&] {
    check_handle(h);
    Level& L = h->levels.back();
    if (!r || !z) throw Error{FEM_E_ARG, "null vector"};
    check_size(nr, L.n_dofs, "r");
    check_size(nz, L.n_dofs, "z");
    const double* dr = in_vec(h, r, nr, 0);
    bool st;
    double* dz = out_vec(h, z, nz, 1, false, &st);
    launch_copy(h, L.b, dr, L.n_dofs);
    vcycle(h, (int)h->levels.size() - 1, L.b, dz);
    finish_out(h, z, dz, nz, st);
  });
}

int fem_rhs(fem_handle h, double* b, int64_t nb) {
  return guarded([&] {
    check_handle(h);
    Level& L = h->levels.back();
    if (!b) throw Error{FEM_E_ARG, "null vector"};
    check_size(nb, L.n_dofs, "b");
    bool st;
    double* db = out_vec(h, b, nb, 0, false, &st);
    launch_zero(h, L.t - L.own_off, L.n_store);
    L.t_zero = false;   // L.t now holds the load vector, not the cleared A x buffer
    launch_rhs(h, L, L.t);
    halo_export_add(h, L, L.t);
    launch_copy(h, db, L.t, L.n_dofs);
    finish_out(h, b, db, nb, st);
  });
}


namespace {
int cg_solve_impl(fem_handle h, const double* b, int64_t nb, double* x, int64_t nx, double rtol,
                  int32_t maxit, int32_t* iters, double* relres, bool zero_start);
}

int cg_solve(fem_handle h, const double* b, int64_t nb, double* x, int64_t nx, double rtol,
             int32_t maxit, int32_t* iters, double* relres) {
  return cg_solve_impl(h, b, nb, x, nx, rtol, maxit, iters, relres, false);
}

int cg_solve_zero(fem_handle h, const double* b, int64_t nb, double* x, int64_t nx, double rtol,
                  int32_t maxit, int32_t* iters, double* relres) {
  return cg_solve_impl(h, b, nb, x, nx, rtol, maxit, iters, relres, true);
}

namespace {
int cg_solve_impl(fem_handle h, const double* b, int64_t nb, double* x, int64_t nx, double rtol,
                  int32_t maxit, int32_t* iters, double* relres, bool zero_start) {
  int result = FEM_OK;
  int rc = guarded([&] {
    check_handle(h);
    Level& L = h->levels.back();
    const int fine = (int)h->levels.size() - 1;
    if (!b || !x) throw Error{FEM_E_ARG, "null vector"};
    check_size(nb, L.n_dofs, "b");
    check_size(nx, L.n_dofs, "x");
    if (!(rtol > 0) || maxit < 0) throw Error{FEM_E_ARG, "rtol must be > 0 and maxit >= 0"};
    const int64_t n = L.n_dofs;
    setup_coarse(h);
    const double* db = in_vec(h, b, nb, 0);
    bool st;
    // zero_start: x is output only (a host x is not uploaded, a device x is cleared here)
    double* dx = out_vec(h, x, nx, 1, !zero_start, &st);
    if (zero_start) launch_zero(h, dx, n);
    if (!L.pcg_r) {
      L.pcg_r = valloc(L);
      L.pcg_p = valloc(L);
      L.pcg_q = valloc(L);
      L.pcg_z = valloc(L);
    }
    double *r = L.pcg_r, *p = L.pcg_p, *q = L.pcg_q, *z = L.pcg_z;
    // CG Dirichlet rows are identity rows: x_c = b_c, r_c = 0 (the system decouples)
    if (is_cg(h)) launch_set_constrained(h, L, db, dx);
    // r_0 = b - A x_0; a zero start (the usual call) skips the operator apply
    dot(h, L, db, db, 6);
    if (!zero_start) dot(h, L, dx, dx, 7);
    FEM_CUDA_TRY(cudaMemcpyAsync(h->hscal, h->scal, sizeof(double) * 8, cudaMemcpyDeviceToHost, h->stream));
    FEM_CUDA_TRY(cudaStreamSynchronize(h->stream));
    if (zero_start || h->hscal[7] == 0.0) {
      launch_copy(h, r, db, n);
      h->hscal[2] = h->hscal[6];
    } else {
      launch_copy(h, p, dx, n);                 // level vector (ghosts) for the first apply
      apply_level(h, L, p, q, true);
      launch_sub(h, r, db, q, n);
      dot(h, L, r, r, 2);
      FEM_CUDA_TRY(cudaMemcpyAsync(h->hscal + 2, h->scal + 2, sizeof(double), cudaMemcpyDeviceToHost, h->stream));
      FEM_CUDA_TRY(cudaStreamSynchronize(h->stream));
    }
    const double bnorm = std::sqrt(h->hscal[6]);
    double rnorm = std::sqrt(h->hscal[2]);
    int it = 0;
    h->hist.assign(1, bnorm > 0 ? rnorm / bnorm : rnorm);
    if (!std::isfinite(rnorm)) throw Error{FEM_E_BREAKDOWN, "non-finite initial residual"};
    // one PCG iteration in two parts
    auto body_pre = [&] {
      vcycle(h, fine, r, z);
      dot(h, L, r, z, 3);
      launch_pcg_update_p(h, p, z, n);      // beta = s3/s0, p = z + beta p, s0 = s3
    };
    auto body_upd = [&] {
      apply_level(h, L, p, q, false, true);
      dot(h, L, p, q, 1);
      launch_pcg_update_xr(h, dx, r, p, q, n);   // alpha = s0/s1, (r,r) -> s2
      if (L.dist) allreduce(h, h->scal + 2, 1);
      FEM_CUDA_TRY(cudaMemcpyAsync(h->hscal, h->scal, sizeof(double) * 4, cudaMemcpyDeviceToHost, h->stream));
    };
    if (rnorm > rtol * bnorm) {
      if (h->use_graphs && (!h->sg.g_pre || h->sg.b != db || h->sg.x != dx)) {
        drop_solve_graphs(h);
        Captured cp = capture(h, h->sg.ev_pre, h->sg.evb_pre, body_pre);
        Captured cu = capture(h, h->sg.ev_upd, h->sg.evb_upd, body_upd);
        h->sg.g_pre = cp.exec;
        h->sg.g_upd = cu.exec;
        h->sg.k_pre = cp.kernels;
        h->sg.k_upd = cu.kernels;
        h->sg.b = db;
        h->sg.x = dx;
        if (std::getenv("FEM_DEBUG"))
          std::fprintf(stderr, "libfem: PCG graphs captured: %lld + %lld kernels per iteration\n",
                       (long long)h->sg.k_pre, (long long)h->sg.k_upd);
      }
      // first iteration through the same code: p = 0 and s0 = 1 make p = z + 0
      launch_zero(h, p, n);
      launch_set_scalar(h, 0, 1.0);
      // the whole loop on the device (conditional WHILE graph, no host round trip per
      // iteration): single rank, no profiling events, FEM_COND_GRAPH != 0
      const char* cge = std::getenv("FEM_COND_GRAPH");
      const bool cond = h->use_graphs && !h->prof.on && !h->comm && maxit < kCondHist && !(cge && std::atoi(cge) == 0);
      if (cond && !h->sg.g_loop) {
        auto upd_nocopy = [&] {
          apply_level(h, L, p, q, false, true);
          dot(h, L, p, q, 1);
          launch_pcg_update_xr(h, dx, r, p, q, n);
        };
        build_cond_loop(h, body_pre, upd_nocopy);
      }
      if (cond && h->sg.g_loop) {
        launch_set_scalar(h, 8, 0.0);
        launch_set_scalar(h, 9, 0.0);
        launch_set_scalar(h, 10, rtol);
        launch_set_scalar(h, 11, (double)maxit);
        FEM_CUDA_TRY(cudaGraphLaunch(h->sg.g_loop, h->stream));
        FEM_CUDA_TRY(cudaMemcpyAsync(h->hscal, h->scal, sizeof(double) * 16, cudaMemcpyDeviceToHost, h->stream));
        FEM_CUDA_TRY(cudaStreamSynchronize(h->stream));
        it = (int)h->hscal[8];
        g_launches += h->sg.k_iter * it;
        std::vector<double> hh(it + 1);
        FEM_CUDA_TRY(cudaMemcpy(hh.data(), h->sg.hist_dev, sizeof(double) * (it + 1), cudaMemcpyDeviceToHost));
        for (int i = 1; i <= it; ++i) h->hist.push_back(hh[i]);
        rnorm = h->hscal[12] * (bnorm > 0 ? bnorm : 1.0);
        if (h->hscal[9] != 0.0)
          throw Error{FEM_E_BREAKDOWN, "PCG breakdown at iteration " + std::to_string(it)};
      }
      while (!(cond && h->sg.g_loop) && it < maxit) {
        if (h->use_graphs) {
          launch_graph(h, h->sg.g_pre, h->sg.k_pre);
          launch_graph(h, h->sg.g_upd, h->sg.k_upd);
        } else {
          body_pre();
          body_upd();
        }
        FEM_CUDA_TRY(cudaStreamSynchronize(h->stream));
        if (h->use_graphs) {
          prof_graph(h, h->sg.ev_pre, h->sg.evb_pre);
          prof_graph(h, h->sg.ev_upd, h->sg.evb_upd);
        }
        ++it;
        if (h->comm) h->comm->check();
        const double pq = h->hscal[1];
        rnorm = std::sqrt(h->hscal[2]);
        h->hist.push_back(bnorm > 0 ? rnorm / bnorm : rnorm);
        if (!(pq > 0) || !std::isfinite(rnorm))
          throw Error{FEM_E_BREAKDOWN, "PCG breakdown at iteration " + std::to_string(it) +
                                           " (p^T A p = " + std::to_string(pq) + ")"};
        if (rnorm <= rtol * bnorm) break;
      }
    }
    if (iters) *iters = it;
    if (relres) *relres = bnorm > 0 ? rnorm / bnorm : rnorm;
    if (rnorm > rtol * bnorm) result = FEM_NOT_CONVERGED;
    finish_out(h, x, dx, nx, st);
    FEM_CUDA_TRY(cudaStreamSynchronize(h->stream));
  });
  return rc != FEM_OK ? rc : result;
}
}  // namespace

int cg_history(fem_handle h, double* rel, int32_t cap, int32_t* n) {
  return guarded([&] {
    check_handle(h);
    if (!rel && cap > 0) throw Error{FEM_E_ARG, "null history buffer"};
    const int32_t m = (int32_t)h->hist.size();
    for (int32_t i = 0; i < std::min(m, cap); ++i) rel[i] = h->hist[i];
    if (n) *n = m;
  });
}

int fem_sync(fem_handle h) {
  return guarded([&] {
    check_handle(h);
    FEM_CUDA_TRY(cudaStreamSynchronize(h->stream));
    if (h->comm) h->comm->check();
  });
}

int fem_profile_read(fem_handle h, double* ms, int64_t* launches, int32_t reset) {
  return fem_profile_read_bytes(h, ms, launches, nullptr, reset);
}

int fem_profile_mode(fem_handle h, int32_t mode) {
  return guarded([&] {
    check_handle(h);
    if (mode < 0 || mode > 2) throw Error{FEM_E_ARG, "profile mode must be 0, 1 or 2"};
    prof_collect(h);
    drop_solve_graphs(h);
    h->prof.on = mode != 0;
    h->prof.mode = mode;
  });
}

int fem_profile_read_bytes(fem_handle h, double* ms, int64_t* launches, double* bytes, int32_t reset) {
  return guarded([&] {
    check_handle(h);
    prof_collect(h);
    if (ms) *ms = h->prof.ms;
    if (launches) *launches = h->prof.launches;
    if (bytes) *bytes = h->prof.bytes;
    if (reset) {
      h->prof.ms = 0;
      h->prof.launches = 0;
      h->prof.bytes = 0;
    }
  });
}

void fem_destroy(fem_handle h) { destroy(h); }

}  // extern "C"
