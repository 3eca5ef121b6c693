// The collectives the sharded paths need, behind one interface (ipt_comm.cu).
//
// Every exchange of the two sharded paths is one of four stream-ordered
// operations, issued by all ranks in the same order:
//   all_reduce  in place (the per-iteration stop scalars, ipt_full.cu / ipt_single.cu)
//   all_gather  in place (Delta's row slices at upload; the single-pair iterate)
//   gather      variable-size blocks to a root (Z column shards, eigenvalues)
//   map_peers   the peer-buffer exchange of the fused all-gather (the map kernel stores
//               its rows of the new iterate straight into every peer's z)
//
// Two backends:
//   NCCL  — one process per GPU (the production path): ncclAllReduce / ncclAllGather /
//           grouped send-recv, peer buffers mapped by CUDA IPC over NVLink.
//   local — several ranks as contexts inside ONE process (one host thread per rank), on
//           one device or several: collectives are host rendezvous + cross-stream event
//           waits + a fixed-order reduction kernel reading every rank's buffer; peer
//           buffers are plain device pointers. No kernel ever waits on another kernel
//           (only stream-ordered event dependencies), so ranks may share one GPU. This
//           drives the library's real multi-rank code (sharded uploads, per-iteration
//           all-reduces, fused peer stores, gathers) on a single B200.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <memory>

namespace iptb {

enum class CommType : int { F64 = 0, I32 = 1, Byte = 2 };
enum class CommOp : int { Sum = 0, Max = 1, Min = 2 };

inline size_t comm_type_size(CommType t) { return t == CommType::F64 ? 8 : t == CommType::I32 ? 4 : 1; }

struct Comm {
  int rank = 0, nranks = 1;
  virtual ~Comm() = default;
  virtual const char* kind() const = 0;
  // buf holds `count` elements on every rank; afterwards every rank holds the same
  // reduction (bitwise identical across ranks).
  virtual void all_reduce(void* buf, size_t count, CommType t, CommOp op, cudaStream_t s) = 0;
  // buf holds nranks blocks of `count` elements; block r is rank r's contribution.
  virtual void all_gather(void* buf, size_t count, CommType t, cudaStream_t s) = 0;
  // Rank r sends `count` elements; the root receives block r at recv + displs[r]
  // (element offsets; counts[r] == rank r's count). recv/counts/displs: root only.
  virtual void gather(const void* send, size_t count, void* recv, const size_t* counts, const size_t* displs,
                      CommType t, int root, cudaStream_t s) = 0;
  // Exchange `nbuf` (<= 2) device buffers of this rank with every peer: peers[b][q] is
  // the q-th other rank's (ascending rank order) buffer b, writable from this device.
  // Returns true on every rank when every rank mapped every peer (false on all otherwise).
  virtual bool map_peers(void* const* mine, int nbuf, void* (*peers)[8], bool* owned_by_ipc) = 0;
  // Mark the group failed (an exception on this rank): ranks blocked in a collective
  // wake up and throw instead of waiting forever.
  virtual void abort() {}
};

struct LocalGroup;
std::unique_ptr<Comm> make_nccl_comm(const void* unique_id128, int rank, int nranks, int device);
std::shared_ptr<LocalGroup> make_local_group(int nranks);
std::unique_ptr<Comm> make_local_comm(const std::shared_ptr<LocalGroup>& g, int rank, int device);
void nccl_unique_id(void* out128);

}  // namespace iptb
