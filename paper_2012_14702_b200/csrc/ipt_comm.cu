// Collective backends of the sharded paths (ipt_comm.cuh): NCCL (one process per GPU)
// and "local" (ranks as contexts of one process, on one device or several).
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <type_traits>
#include <vector>

#include "ipt_internal.cuh"

namespace iptb {

namespace {

void nccl_check(ncclResult_t r, const char* what, const char* file, int line) {
  if (r != ncclSuccess)
    throw NcclError(std::string("NCCL error ") + ncclGetErrorString(r) + " in " + what + " at " + file + ":" +
                    std::to_string(line));
}
#define IPT_NCCL(x) nccl_check((x), #x, __FILE__, __LINE__)

ncclDataType_t nccl_type(CommType t) {
  return t == CommType::F64 ? ncclDouble : t == CommType::I32 ? ncclInt32 : ncclChar;
}
ncclRedOp_t nccl_op(CommOp o) { return o == CommOp::Sum ? ncclSum : o == CommOp::Max ? ncclMax : ncclMin; }

// ------------------------------------------------------------------ NCCL backend

struct NcclComm final : Comm {
  ncclComm_t comm = nullptr;
  int device = 0;
  ~NcclComm() override {
    if (comm) ncclCommDestroy(comm);
  }
  const char* kind() const override { return "nccl"; }

  void all_reduce(void* buf, size_t count, CommType t, CommOp op, cudaStream_t s) override {
    NvtxRange nvtx_("ipt:all_reduce");
    IPT_NCCL(ncclAllReduce(buf, buf, count, nccl_type(t), nccl_op(op), comm, s));
  }
  void all_gather(void* buf, size_t count, CommType t, cudaStream_t s) override {
    NvtxRange nvtx_("ipt:all_gather");
    char* b = static_cast<char*>(buf);
    IPT_NCCL(ncclAllGather(b + size_t(rank) * count * comm_type_size(t), b, count, nccl_type(t), comm, s));
  }
  void gather(const void* send, size_t count, void* recv, const size_t* counts, const size_t* displs, CommType t,
              int root, cudaStream_t s) override {
    NvtxRange nvtx_("ipt:gather");
    const size_t sz = comm_type_size(t);
    IPT_NCCL(ncclGroupStart());
    if (rank == root) {
      for (int r = 0; r < nranks; ++r) {
        if (counts[r] == 0) continue;
        char* dst = static_cast<char*>(recv) + displs[r] * sz;
        if (r == root)
          IPT_CUDA(cudaMemcpyAsync(dst, send, counts[r] * sz, cudaMemcpyDeviceToDevice, s));
        else
          IPT_NCCL(ncclRecv(dst, counts[r], nccl_type(t), r, comm, s));
      }
    } else if (count > 0) {
      IPT_NCCL(ncclSend(send, count, nccl_type(t), root, comm, s));
    }
    IPT_NCCL(ncclGroupEnd());
  }
  // CUDA IPC handles all-gathered over the communicator; the outcome agreed by a min
  // all-reduce (if any rank cannot map a peer, none uses peer stores).
  bool map_peers(void* const* mine, int nbuf, void* (*peers)[8], bool* owned_by_ipc) override {
    struct Handles {
      cudaIpcMemHandle_t h[2];
    };
    Handles me{};
    int ok = 1;
    for (int b = 0; b < nbuf; ++b)
      if (cudaIpcGetMemHandle(&me.h[b], mine[b]) != cudaSuccess) ok = 0;
    cudaGetLastError();
    const size_t hb = sizeof(Handles);
    char* dv = nullptr;
    IPT_CUDA(cudaMalloc(&dv, hb * nranks + 64));
    cudaStream_t s = nullptr;
    IPT_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    IPT_CUDA(cudaMemcpyAsync(dv + hb * rank, &me, hb, cudaMemcpyHostToDevice, s));
    all_gather(dv, hb, CommType::Byte, s);
    std::vector<Handles> all(nranks);
    IPT_CUDA(cudaMemcpyAsync(all.data(), dv, hb * nranks, cudaMemcpyDeviceToHost, s));
    IPT_CUDA(cudaStreamSynchronize(s));
    int q = 0;
    for (int r = 0; r < nranks && ok; ++r) {
      if (r == rank) continue;
      for (int b = 0; b < nbuf && ok; ++b) {
        void* ptr = nullptr;
        if (cudaIpcOpenMemHandle(&ptr, all[r].h[b], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
          cudaGetLastError();
          ok = 0;
        } else {
          peers[b][q] = ptr;
        }
      }
      ++q;
    }
    int* dok = reinterpret_cast<int*>(dv + hb * nranks);
    IPT_CUDA(cudaMemcpyAsync(dok, &ok, sizeof(int), cudaMemcpyHostToDevice, s));
    all_reduce(dok, 1, CommType::I32, CommOp::Min, s);
    int all_ok = 0;
    IPT_CUDA(cudaMemcpyAsync(&all_ok, dok, sizeof(int), cudaMemcpyDeviceToHost, s));
    IPT_CUDA(cudaStreamSynchronize(s));
    cudaStreamDestroy(s);
    cudaFree(dv);
    *owned_by_ipc = true;
    if (!all_ok) {
      for (int b = 0; b < nbuf; ++b)
        for (int k = 0; k < 8; ++k)
          if (peers[b][k]) {
            cudaIpcCloseMemHandle(peers[b][k]);
            peers[b][k] = nullptr;
          }
    }
    return all_ok != 0;
  }
};

// ------------------------------------------------------------------ local backend

constexpr int kMaxLocalRanks = 16;

struct LocalPtrs {
  const void* p[kMaxLocalRanks];
};

// Fixed rank order 0..nr-1 on every rank: the result is bitwise identical everywhere.
template <typename T>
__global__ void local_reduce_kernel(LocalPtrs src, int nr, T* __restrict__ dst, size_t count, int op) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < count; i += size_t(gridDim.x) * blockDim.x) {
    T acc = static_cast<const T*>(src.p[0])[i];
    for (int r = 1; r < nr; ++r) {
      const T v = static_cast<const T*>(src.p[r])[i];
      if (op == 0) acc = acc + v;
      else if constexpr (std::is_same<T, double>::value) acc = op == 1 ? nan_max(acc, v) : -nan_max(-acc, -v);
      else acc = op == 1 ? (v > acc ? v : acc) : (v < acc ? v : acc);
    }
    dst[i] = acc;
  }
}

}  // namespace

struct LocalGroup {
  int nranks = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  bool aborted = false;
  int joined = 0;
  double timeout_s = 600.0;
  // per-rank slots (written before the first rendezvous of an operation, read between
  // its first and second rendezvous)
  const void* ptr[kMaxLocalRanks] = {};
  void* bufs[kMaxLocalRanks][2] = {};
  int flag[kMaxLocalRanks] = {};
  int device[kMaxLocalRanks] = {};
  cudaEvent_t ready[kMaxLocalRanks] = {};
  cudaEvent_t done[kMaxLocalRanks] = {};

  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    if (aborted) throw CommAborted("local comm: group aborted by another rank");
    const uint64_t g = gen;
    if (++arrived == nranks) {
      arrived = 0;
      ++gen;
      cv.notify_all();
      return;
    }
    const bool woke = cv.wait_for(lk, std::chrono::duration<double>(timeout_s), [&] { return gen != g || aborted; });
    if (!woke) {
      aborted = true;
      cv.notify_all();
      throw CommAborted("local comm: rendezvous timed out (a rank did not reach the collective)");
    }
    if (gen == g) throw CommAborted("local comm: group aborted by another rank");
  }
  void abort() {
    std::lock_guard<std::mutex> lk(mu);
    aborted = true;
    cv.notify_all();
  }
};

namespace {

struct LocalComm final : Comm {
  std::shared_ptr<LocalGroup> G;
  int device = 0;
  void* scratch = nullptr;
  size_t scratch_bytes = 0;

  ~LocalComm() override {
    DeviceGuard dg(device);
    if (G->ready[rank]) cudaEventDestroy(G->ready[rank]);
    if (G->done[rank]) cudaEventDestroy(G->done[rank]);
    G->ready[rank] = G->done[rank] = nullptr;
    if (scratch) cudaFree(scratch);
  }
  const char* kind() const override { return "local"; }
  void abort() override { G->abort(); }

  void post(const void* p, cudaStream_t s) {
    G->ptr[rank] = p;
    IPT_CUDA(cudaEventRecord(G->ready[rank], s));
    G->barrier();
  }
  void wait_peers(cudaEvent_t* evs, cudaStream_t s) {
    for (int p = 0; p < nranks; ++p)
      if (p != rank) IPT_CUDA(cudaStreamWaitEvent(s, evs[p], 0));
  }
  void finish(cudaStream_t s, bool wait_all, int only = -1) {
    IPT_CUDA(cudaEventRecord(G->done[rank], s));
    G->barrier();
    if (wait_all) wait_peers(G->done, s);
    else if (only >= 0 && only != rank) IPT_CUDA(cudaStreamWaitEvent(s, G->done[only], 0));
  }

  void all_reduce(void* buf, size_t count, CommType t, CommOp op, cudaStream_t s) override {
    NvtxRange nvtx_("ipt:all_reduce");
    if (t == CommType::Byte) throw InvalidArgument("local comm: byte all-reduce");
    const size_t bytes = count * comm_type_size(t);
    if (bytes > scratch_bytes) {
      if (scratch) {
        IPT_CUDA(cudaStreamSynchronize(s));
        cudaFree(scratch);
      }
      scratch_bytes = std::max<size_t>(bytes, 4096);
      IPT_CUDA(cudaMalloc(&scratch, scratch_bytes));
    }
    post(buf, s);
    wait_peers(G->ready, s);
    LocalPtrs src{};
    for (int p = 0; p < nranks; ++p) src.p[p] = G->ptr[p];
    const unsigned grid = static_cast<unsigned>(std::min<size_t>(ceil_div(int64_t(count), 256), 1184));
    if (grid) {
      if (t == CommType::F64)
        local_reduce_kernel<double><<<grid, 256, 0, s>>>(src, nranks, static_cast<double*>(scratch), count, int(op));
      else
        local_reduce_kernel<int32_t><<<grid, 256, 0, s>>>(src, nranks, static_cast<int32_t*>(scratch), count, int(op));
      IPT_LAUNCH_CHECK();
      count_launch();
    }
    finish(s, true);  // every rank's reads of `buf` done before anyone overwrites it
    if (bytes) IPT_CUDA(cudaMemcpyAsync(buf, scratch, bytes, cudaMemcpyDeviceToDevice, s));
  }

  void all_gather(void* buf, size_t count, CommType t, cudaStream_t s) override {
    NvtxRange nvtx_("ipt:all_gather");
    const size_t bytes = count * comm_type_size(t);
    post(buf, s);
    wait_peers(G->ready, s);
    for (int p = 0; p < nranks; ++p) {
      if (p == rank || bytes == 0) continue;
      IPT_CUDA(cudaMemcpyAsync(static_cast<char*>(buf) + p * bytes, static_cast<const char*>(G->ptr[p]) + p * bytes,
                               bytes, cudaMemcpyDefault, s));
    }
    finish(s, true);
  }

  void gather(const void* send, size_t count, void* recv, const size_t* counts, const size_t* displs, CommType t,
              int root, cudaStream_t s) override {
    NvtxRange nvtx_("ipt:gather");
    const size_t sz = comm_type_size(t);
    (void)count;
    post(send, s);
    if (rank == root) {
      wait_peers(G->ready, s);
      for (int p = 0; p < nranks; ++p) {
        if (counts[p] == 0) continue;
        IPT_CUDA(cudaMemcpyAsync(static_cast<char*>(recv) + displs[p] * sz, G->ptr[p], counts[p] * sz,
                                 cudaMemcpyDefault, s));
      }
    }
    finish(s, false, root);  // senders keep their buffers until the root has copied them
  }

  bool map_peers(void* const* mine, int nbuf, void* (*peers)[8], bool* owned_by_ipc) override {
    for (int b = 0; b < nbuf; ++b) G->bufs[rank][b] = mine[b];
    G->barrier();
    int ok = 1, q = 0;
    for (int p = 0; p < nranks; ++p) {
      if (p == rank) continue;
      if (G->device[p] != device) {
        int can = 0;
        cudaDeviceCanAccessPeer(&can, device, G->device[p]);
        if (!can) ok = 0;
      }
      for (int b = 0; b < nbuf; ++b) peers[b][q] = G->bufs[p][b];
      ++q;
    }
    G->flag[rank] = ok;
    G->barrier();
    int all_ok = 1;
    for (int p = 0; p < nranks; ++p) all_ok &= G->flag[p];
    G->barrier();
    *owned_by_ipc = false;
    if (!all_ok)
      for (int b = 0; b < nbuf; ++b)
        for (int k = 0; k < 8; ++k) peers[b][k] = nullptr;
    return all_ok != 0;
  }
};

}  // namespace

std::unique_ptr<Comm> make_nccl_comm(const void* unique_id128, int rank, int nranks, int device) {
  auto c = std::make_unique<NcclComm>();
  c->rank = rank;
  c->nranks = nranks;
  c->device = device;
  ncclUniqueId id;
  std::memcpy(&id, unique_id128, sizeof(id));
  IPT_NCCL(ncclCommInitRank(&c->comm, nranks, id, rank));
  return c;
}

void nccl_unique_id(void* out128) {
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId id;
  IPT_NCCL(ncclGetUniqueId(&id));
  std::memcpy(out128, &id, sizeof(id));
}

std::shared_ptr<LocalGroup> make_local_group(int nranks) {
  if (nranks < 1 || nranks > kMaxLocalRanks) throw InvalidArgument("local comm: 1..16 ranks");
  auto g = std::make_shared<LocalGroup>();
  g->nranks = nranks;
  if (const char* e = std::getenv("IPT_LOCAL_COMM_TIMEOUT_S")) g->timeout_s = std::max(1.0, std::atof(e));
  return g;
}

std::unique_ptr<Comm> make_local_comm(const std::shared_ptr<LocalGroup>& g, int rank, int device) {
  if (!g || rank < 0 || rank >= g->nranks) throw InvalidArgument("local comm: bad rank");
  auto c = std::make_unique<LocalComm>();
  c->G = g;
  c->rank = rank;
  c->nranks = g->nranks;
  c->device = device;
  DeviceGuard dg(device);
  {
    std::lock_guard<std::mutex> lk(g->mu);
    if (g->ready[rank]) throw InvalidArgument("local comm: rank already joined");
    IPT_CUDA(cudaEventCreateWithFlags(&g->ready[rank], cudaEventDisableTiming));
    IPT_CUDA(cudaEventCreateWithFlags(&g->done[rank], cudaEventDisableTiming));
    g->device[rank] = device;
    ++g->joined;
  }
  // ranks on other devices of this process read and write each other's buffers directly
  for (int d = 0; d < 64; ++d) {
    int count = 0;
    cudaGetDeviceCount(&count);
    if (d >= count) break;
    if (d == device) continue;
    int can = 0;
    if (cudaDeviceCanAccessPeer(&can, device, d) == cudaSuccess && can) {
      const cudaError_t e = cudaDeviceEnablePeerAccess(d, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) throw CudaError("local comm: peer access");
      cudaGetLastError();
      // the library's buffers come from the stream-ordered pool: grant device d access to
      // this device's pool (the collectives read peers' buffers directly)
      cudaMemPool_t pool;
      if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        cudaMemAccessDesc desc{};
        desc.location.type = cudaMemLocationTypeDevice;
        desc.location.id = d;
        desc.flags = cudaMemAccessFlagsProtReadWrite;
        IPT_CUDA(cudaMemPoolSetAccess(pool, &desc, 1));
      }
    }
  }
  return c;
}

}  // namespace iptb
