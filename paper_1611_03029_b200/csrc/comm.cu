// Transports of the z-slab exchanges (include/fem.h "multi-rank").
//
// NcclComm: one process per GPU.  NCCL is resolved at run time with dlopen of
// libnccl.so.2 (a copy the process has already loaded, e.g. torch's, is reused),
// so libfem loads without NCCL on single-GPU hosts.  Exchanges are grouped
// ncclSend/ncclRecv, reductions ncclAllReduce, all on the caller's stream (so they
// can be captured into the PCG CUDA graphs).
//
// LocalComm: nranks threads of one process sharing one device (tests; running
// the multi-rank path on one GPU).  A collective is two host barriers: every
// rank records a "ready" event after the data it offers, then each rank pulls
// what it needs with device-to-device copies ordered after the owner's event,
// records "done", and before continuing waits for the "done" events of the ranks
// that read its buffers.  No kernel ever waits on another: all ordering is
// stream/event dependencies known when the work is enqueued.
#include <dlfcn.h>
#include <nccl.h>

#include <chrono>
#include <condition_variable>
#include <cstring>
#include <mutex>

#include "internal.h"

namespace fem {

// ---------------------------------------------------------------- NCCL
namespace {

struct NcclApi {
  void* so = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* so = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!so) so = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!so) so = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!so) return;
    api.so = so;
#define FEM_NCCL_SYM(f) api.f = reinterpret_cast<decltype(api.f)>(dlsym(so, "nccl" #f))
    FEM_NCCL_SYM(GetUniqueId);
    FEM_NCCL_SYM(CommInitRank);
    FEM_NCCL_SYM(CommDestroy);
    FEM_NCCL_SYM(Send);
    FEM_NCCL_SYM(Recv);
    FEM_NCCL_SYM(AllReduce);
    FEM_NCCL_SYM(GroupStart);
    FEM_NCCL_SYM(GroupEnd);
    FEM_NCCL_SYM(GetErrorString);
    FEM_NCCL_SYM(CommGetAsyncError);
#undef FEM_NCCL_SYM
  });
  if (!api.so || !api.GetUniqueId || !api.CommInitRank || !api.Send || !api.Recv || !api.AllReduce ||
      !api.GroupStart || !api.GroupEnd)
    throw Error{FEM_E_NCCL, "libnccl.so.2 could not be loaded (multi-rank needs NCCL)"};
  return api;
}

void nccl_try(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) {
    const char* m = nccl().GetErrorString ? nccl().GetErrorString(r) : "?";
    throw Error{FEM_E_NCCL, std::string(what) + ": " + m};
  }
}

class NcclComm : public Comm {
 public:
  NcclComm(const void* id, int r, int p) {
    rank = r;
    nranks = p;
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    nccl_try(nccl().CommInitRank(&comm_, p, uid, r), "ncclCommInitRank");
  }
  ~NcclComm() override {
    if (comm_ && nccl().CommDestroy) nccl().CommDestroy(comm_);
  }
  void exchange(const std::vector<Msg>& sends, const std::vector<Msg>& recvs, cudaStream_t s) override {
    if (sends.empty() && recvs.empty()) return;
    nccl_try(nccl().GroupStart(), "ncclGroupStart");
    for (const auto& m : sends) nccl_try(nccl().Send(m.ptr, (size_t)m.n, ncclFloat64, m.peer, comm_, s), "ncclSend");
    for (const auto& m : recvs) nccl_try(nccl().Recv(m.ptr, (size_t)m.n, ncclFloat64, m.peer, comm_, s), "ncclRecv");
    nccl_try(nccl().GroupEnd(), "ncclGroupEnd");
  }
  void allreduce_sum(double* p, int64_t n, cudaStream_t s) override {
    nccl_try(nccl().AllReduce(p, p, (size_t)n, ncclFloat64, ncclSum, comm_, s), "ncclAllReduce");
  }
  bool graph_capturable() const override { return true; }
  // a peer that died or a network fault surfaces here instead of as a hang in the next
  // synchronisation (polled after every PCG iteration and in fem_sync)
  void check() override {
    if (!nccl().CommGetAsyncError) return;
    ncclResult_t st = ncclSuccess;
    nccl_try(nccl().CommGetAsyncError(comm_, &st), "ncclCommGetAsyncError");
    if (st != ncclSuccess && st != ncclInProgress) nccl_try(st, "NCCL asynchronous error");
  }

 private:
  ncclComm_t comm_ = nullptr;
};

// ---------------------------------------------------------------- in-process group
constexpr int kMaxLocalRanks = 16;

struct PtrSet {
  const double* p[kMaxLocalRanks];
};

// out[i] = sum over ranks j (in rank order, so every rank gets the same bits) of in_j[i]
__global__ void sum_ranks_kernel(double* __restrict__ out, PtrSet in, int P, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int j = 0; j < P; ++j) s += in.p[j][i];
    out[i] = s;
  }
}

struct LocalGroup {
  explicit LocalGroup(int p) : P(p), posted(p), red(p, nullptr), ready(p, nullptr), done(p, nullptr) {}
  int P;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  struct Posted {
    int dst, tag;
    const double* ptr;
    int64_t n;
  };
  std::vector<std::vector<Posted>> posted;   // per source rank
  std::vector<const double*> red;            // allreduce inputs per rank
  std::vector<cudaEvent_t> ready, done;      // per rank (created by the rank's thread)

  void barrier() {
    std::unique_lock<std::mutex> lk(m);
    const uint64_t g = gen;
    if (++arrived == P) {
      arrived = 0;
      ++gen;
      cv.notify_all();
      return;
    }
    if (!cv.wait_for(lk, std::chrono::seconds(300), [&] { return gen != g; }))
      throw Error{FEM_E_NCCL, "in-process group: barrier timed out (a rank did not enter the collective)"};
  }
};

class LocalComm : public Comm {
 public:
  LocalComm(LocalGroup* g, int r, int p) : g_(g) {
    rank = r;
    nranks = p;
    FEM_CUDA_TRY(cudaEventCreateWithFlags(&g_->ready[r], cudaEventDisableTiming));
    FEM_CUDA_TRY(cudaEventCreateWithFlags(&g_->done[r], cudaEventDisableTiming));
  }
  ~LocalComm() override {
    cudaEventDestroy(g_->ready[rank]);
    cudaEventDestroy(g_->done[rank]);
    if (tmp_) cudaFree(tmp_);
  }
  void exchange(const std::vector<Msg>& sends, const std::vector<Msg>& recvs, cudaStream_t s) override {
    {
      std::lock_guard<std::mutex> lk(g_->m);
      auto& mine = g_->posted[rank];
      mine.clear();
      for (const auto& m : sends) mine.push_back({m.peer, m.tag, m.ptr, m.n});
    }
    FEM_CUDA_TRY(cudaEventRecord(g_->ready[rank], s));
    g_->barrier();
    for (const auto& m : recvs) {
      const LocalGroup::Posted* src = nullptr;
      for (const auto& q : g_->posted[m.peer])
        if (q.dst == rank && q.tag == m.tag) src = &q;
      if (!src || src->n != m.n)
        throw Error{FEM_E_NCCL, "in-process group: unmatched receive from rank " + std::to_string(m.peer)};
      FEM_CUDA_TRY(cudaStreamWaitEvent(s, g_->ready[m.peer], 0));
      FEM_CUDA_TRY(cudaMemcpyAsync(m.ptr, src->ptr, sizeof(double) * m.n, cudaMemcpyDeviceToDevice, s));
    }
    FEM_CUDA_TRY(cudaEventRecord(g_->done[rank], s));
    g_->barrier();
    for (const auto& m : sends) FEM_CUDA_TRY(cudaStreamWaitEvent(s, g_->done[m.peer], 0));
    g_->barrier();   // the posted table may be rewritten by the next collective
  }
  void allreduce_sum(double* p, int64_t n, cudaStream_t s) override {
    if (tmp_n_ < n) {
      if (tmp_) cudaFree(tmp_);
      FEM_CUDA_TRY(cudaMalloc(&tmp_, sizeof(double) * n));
      tmp_n_ = n;
    }
    g_->red[rank] = p;
    FEM_CUDA_TRY(cudaEventRecord(g_->ready[rank], s));
    g_->barrier();
    PtrSet in;
    for (int j = 0; j < nranks; ++j) {
      in.p[j] = g_->red[j];
      if (j != rank) FEM_CUDA_TRY(cudaStreamWaitEvent(s, g_->ready[j], 0));
    }
    const unsigned grid = (unsigned)std::min<int64_t>((n + 255) / 256, 1184);
    sum_ranks_kernel<<<grid, 256, 0, s>>>(tmp_, in, nranks, n);
    count_launch();
    check_launch("sum_ranks_kernel");
    FEM_CUDA_TRY(cudaEventRecord(g_->done[rank], s));
    g_->barrier();
    for (int j = 0; j < nranks; ++j)
      if (j != rank) FEM_CUDA_TRY(cudaStreamWaitEvent(s, g_->done[j], 0));
    FEM_CUDA_TRY(cudaMemcpyAsync(p, tmp_, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
    g_->barrier();
  }
  bool graph_capturable() const override { return false; }

 private:
  LocalGroup* g_;
  double* tmp_ = nullptr;
  int64_t tmp_n_ = 0;
};

}  // namespace

std::unique_ptr<Comm> make_nccl_comm(const void* id, int rank, int nranks) {
  return std::unique_ptr<Comm>(new NcclComm(id, rank, nranks));
}

std::unique_ptr<Comm> make_local_comm(void* group, int rank, int nranks) {
  auto* g = static_cast<LocalGroup*>(group);
  if (g->P != nranks) throw Error{FEM_E_ARG, "local group size differs from mesh.nranks"};
  return std::unique_ptr<Comm>(new LocalComm(g, rank, nranks));
}

}  // namespace fem

extern "C" {

int fem_nccl_unique_id(void* id, int64_t len) {
  try {
    if (!id || len < (int64_t)sizeof(ncclUniqueId)) throw fem::Error{FEM_E_ARG, "id buffer must hold 128 bytes"};
    ncclUniqueId uid;
    fem::nccl_try(fem::nccl().GetUniqueId(&uid), "ncclGetUniqueId");
    std::memcpy(id, &uid, sizeof(uid));
    return FEM_OK;
  } catch (const fem::Error& e) {
    fem::set_error(e.msg);
    return e.code;
  }
}

int fem_local_group_create(int32_t nranks, void** group) {
  if (!group || nranks < 1 || nranks > fem::kMaxLocalRanks) {
    fem::set_error("nranks must be in [1, 16] and group non-null");
    return FEM_E_ARG;
  }
  *group = new fem::LocalGroup(nranks);
  return FEM_OK;
}

void fem_local_group_destroy(void* group) { delete static_cast<fem::LocalGroup*>(group); }

}  // extern "C"
