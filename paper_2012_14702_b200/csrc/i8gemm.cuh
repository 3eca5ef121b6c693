// 5th-generation tensor-core INT8 GEMM for sm_100a (tcgen05.mma kind::i8, int32 TMEM
// accumulators): the building block of FP64-accurate products by modular integer
// arithmetic (Ozaki scheme II, see ozaki.cu). tcgen05 has no f64 kind; exact integer
// products on the INT8 datapath are how FP64 GEMMs use the 5th-gen tensor cores.
//
// C[m, n] = sum_k A[m, k] * B[n, k]     A: M x K int8 (K contiguous), B: N x K int8 (K
// contiguous), exact int32 accumulation (|sum| < K * 2^14 for residues in [-128, 127]).
//
// CTA tile 128 x 256 x 128 bytes, 4-stage TMA pipeline (SWIZZLE_128B, 48 KB per stage),
// warp roles: warp 0 issues TMA, warp 1 allocates 256 TMEM columns and one elected lane
// issues 4 tcgen05.mma (K = 32 each) per stage, committing stage release and accumulator
// completion to mbarriers; warps 2-5 drain TMEM (tcgen05.ld 32x32b) in the epilogue. The
// epilogue is a functor applied to each row's 32-column chunk of int32 results.
#pragma once

#include <cstdlib>
#include <string>

#include "dmma_gemm.cuh"
#include "ipt_internal.cuh"

namespace iptb {

constexpr int kI8BM = 128;
constexpr int kI8BN = 256;
constexpr int kI8BK = 128;  // bytes = int8 elements per stage along K
constexpr int kI8Stages = 4;
constexpr int kI8Threads = 192;  // 6 warps
constexpr int kI8Threads2 = 256;  // cta_group::2 kernels: 8 warps, all of them drain TMEM in the epilogue
constexpr int kI8StageBytes = (kI8BM + kI8BN) * kI8BK;
constexpr size_t kI8SmemBytes = size_t(kI8Stages) * kI8StageBytes + 1024 + 256;

__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t smem_addr) {
  // SM100 shared-memory matrix descriptor, K-major, 128-byte swizzle: start address
  // (>> 4), LBO unused (1), SBO = 1024 B between 8-row core-matrix groups, version 1.
  uint64_t d = 0;
  d |= uint64_t((smem_addr & 0x3FFFF) >> 4);
  d |= uint64_t(1) << 16;
  d |= uint64_t(1024 >> 4) << 32;
  d |= uint64_t(1) << 46;
  d |= uint64_t(2) << 61;
  return d;
}

__device__ __forceinline__ void umma_i8(uint32_t tmem_c, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, {%5, %6, %7, %8}, p;\n\t}\n" ::"r"(tmem_c),
      "l"(da), "l"(db), "r"(idesc), "r"(acc), "r"(0u), "r"(0u), "r"(0u), "r"(0u));
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
        "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// instruction descriptor: int32 accumulate, signed int8 A and B, both K-major, M = 128, N = 256
constexpr uint32_t kI8Idesc = (2u << 4) | (1u << 7) | (1u << 10) | (uint32_t(kI8BN >> 3) << 17) |
                              (uint32_t(kI8BM >> 4) << 24);

// Grouped rasterisation: `group` consecutive M tiles sweep the N tiles together, so the
// CTAs resident at one time share both their A and their B tiles in L2 (M-fastest order
// over all of M re-streams A from DRAM once per N tile).
__device__ __forceinline__ void grouped_tile(int t, int tiles_m, int tiles_n, int group, int& tm, int& tn) {
  const int per_group = group * tiles_n;
  const int g = t / per_group, first = g * group;
  const int gs = min(group, tiles_m - first);
  const int r = t - g * per_group;
  tm = first + r % gs;
  tn = r / gs;
}

// Epi(row, col0, v[32]) consumes columns col0..col0+31 of one row; Epi::skip() (read once,
// uniform) lets a launch exit before any setup.
template <class Epi>
__global__ void __launch_bounds__(kI8Threads, 1)
    i8gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int K, int tiles_m,
                  int tiles_n, int group, Epi epi) {
  if (epi.skip()) return;  // uniform over the grid (e.g. an unused Ozaki modulus)
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(base + size_t(kI8Stages) * kI8StageBytes);
  uint64_t* empty = full + kI8Stages;
  uint64_t* acc_full = empty + kI8Stages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_full + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int tm, tn;
  grouped_tile(blockIdx.x, tiles_m, tiles_n, group, tm, tn);
  const int m0 = tm * kI8BM, n0 = tn * kI8BN;
  const int KB = K / kI8BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kI8Stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(acc_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(uint32_t(kI8BN)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tmA) : "memory");
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tmB) : "memory");
      for (int kb = 0; kb < KB; ++kb) {
        const int s = kb % kI8Stages;
        if (kb >= kI8Stages) mbar_wait(&empty[s], ((kb / kI8Stages) - 1) & 1);
        unsigned char* sa = base + size_t(s) * kI8StageBytes;
        mbar_expect_tx(&full[s], kI8StageBytes);
        tma_load_2d(sa, &tmA, &full[s], kb * kI8BK, m0);
        tma_load_2d(sa + kI8BM * kI8BK, &tmB, &full[s], kb * kI8BK, n0);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      for (int kb = 0; kb < KB; ++kb) {
        const int s = kb % kI8Stages;
        mbar_wait(&full[s], (kb / kI8Stages) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t sa = smem_u32(base + size_t(s) * kI8StageBytes);
        const uint64_t da = umma_desc_sw128(sa), db = umma_desc_sw128(sa + kI8BM * kI8BK);
#pragma unroll
        for (int k = 0; k < kI8BK / 32; ++k)  // 32 bytes of K per MMA: +2 in the (>>4) start field
          umma_i8(tmem, da + 2 * k, db + 2 * k, kI8Idesc, (kb | k) ? 1u : 0u);
        umma_commit(&empty[s]);
      }
      umma_commit(acc_full);
    }
    __syncwarp();
  } else {
    // epilogue: warp w reads TMEM lanes 32*(w%4) .. +31 (its rows), 32 columns at a time
    mbar_wait(acc_full, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int quarter = warp & 3;
    const int row = m0 + quarter * 32 + lane;
    const uint32_t trow = tmem + (uint32_t(quarter * 32) << 16);
#pragma unroll 1
    for (int c = 0; c < kI8BN; c += 32) {
      uint32_t v[32];
      tmem_ld32(trow + uint32_t(c), v);
      epi(row, n0 + c, v);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(uint32_t(kI8BN)));
}

// ---- 2-CTA cluster variant: the two CTAs of a cluster own vertically adjacent 128-row
// tiles with the same 256 columns and share the B tile: each loads one 128-row half of
// it with a cluster-multicast TMA into both CTAs' shared memory, and each MMA completion
// is committed to both CTAs' stage barriers. L2->SM operand traffic per output drops by
// a third (the single-CTA kernel is L2-bandwidth bound). ----
__device__ __forceinline__ void tma_load_2d_mc(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y,
                                               uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%3, %4}], [%2], %5;\n" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(x), "r"(y), "h"(mask)
      : "memory");
}

__device__ __forceinline__ void umma_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <class Epi>
__global__ void __launch_bounds__(kI8Threads, 1)
    i8gemm_mc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int K,
                     int tiles_m, int tiles_n, int group, Epi epi) {
  if (epi.skip()) return;  // uniform over the grid (e.g. an unused Ozaki modulus)
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(base + size_t(kI8Stages) * kI8StageBytes);
  uint64_t* empty = full + kI8Stages;
  uint64_t* acc_full = empty + kI8Stages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_full + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rank = static_cast<int>(cluster_rank());
  const int pairs_m = tiles_m / 2;
  const int cl = blockIdx.x >> 1;
  int pm, tn;
  grouped_tile(cl, pairs_m, tiles_n, group, pm, tn);
  const int tm = 2 * pm + rank;
  const int m0 = tm * kI8BM, n0 = tn * kI8BN;
  const int KB = K / kI8BK;
  constexpr uint16_t kBoth = 0x3;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kI8Stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 2);  // this CTA's MMA and the peer's both read stage s
    }
    mbar_init(acc_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(uint32_t(kI8BN)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync_all();  // the peer's barriers exist before anything is multicast to them
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tmA) : "memory");
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tmB) : "memory");
      for (int kb = 0; kb < KB; ++kb) {
        const int s = kb % kI8Stages;
        if (kb >= kI8Stages) mbar_wait(&empty[s], ((kb / kI8Stages) - 1) & 1);
        unsigned char* sa = base + size_t(s) * kI8StageBytes;
        mbar_expect_tx(&full[s], kI8StageBytes);  // own A + both halves of B
        tma_load_2d(sa, &tmA, &full[s], kb * kI8BK, m0);
        tma_load_2d_mc(sa + kI8BM * kI8BK + rank * (kI8BN / 2) * kI8BK, &tmB, &full[s], kb * kI8BK,
                       n0 + rank * (kI8BN / 2), kBoth);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      for (int kb = 0; kb < KB; ++kb) {
        const int s = kb % kI8Stages;
        mbar_wait(&full[s], (kb / kI8Stages) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t sa = smem_u32(base + size_t(s) * kI8StageBytes);
        const uint64_t da = umma_desc_sw128(sa), db = umma_desc_sw128(sa + kI8BM * kI8BK);
#pragma unroll
        for (int k = 0; k < kI8BK / 32; ++k)
          umma_i8(tmem, da + 2 * k, db + 2 * k, kI8Idesc, (kb | k) ? 1u : 0u);
        umma_commit_mc(&empty[s], kBoth);
      }
      umma_commit(acc_full);
    }
    __syncwarp();
  } else {
    mbar_wait(acc_full, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int quarter = warp & 3;
    const int row = m0 + quarter * 32 + lane;
    const uint32_t trow = tmem + (uint32_t(quarter * 32) << 16);
#pragma unroll 1
    for (int c = 0; c < kI8BN; c += 32) {
      uint32_t v[32];
      tmem_ld32(trow + uint32_t(c), v);
      epi(row, n0 + c, v);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(uint32_t(kI8BN)));
  cluster_sync_all();  // no CTA leaves while the peer may still signal its barriers
}

// ---- 2-SM MMA variant (tcgen05.mma.cta_group::2): the CTA pair of a cluster computes a
// 256 x 256 tile; each CTA stages its 128 rows of A and its 128 rows of B (32 KB per
// k-block, 6 stages), the leader CTA issues M = 256 MMAs that read both CTAs' shared
// memory and write each CTA's 128 accumulator lanes in its own TMEM. Both producers'
// TMA bytes complete on the leader's stage barrier; the leader's MMA commits release the
// stage in both CTAs and signal both epilogues. ----
// NB = 1: 256 x 256 tile per pair; NB = 2: 256 x 512 (two N = 256 MMAs share the A tile,
// all 512 TMEM columns), which cuts the operand bytes per MAC by a further quarter.
template <int NB>
struct I8S2 {
  static constexpr int kStages = NB == 1 ? 6 : 4;
  static constexpr int kStageBytes = (1 + NB) * 128 * kI8BK;  // own A rows + own B rows
  static constexpr size_t kSmem = size_t(kStages) * kStageBytes + 1024 + 256;
};
constexpr uint32_t kI8Idesc2 = (2u << 4) | (1u << 7) | (1u << 10) | (uint32_t(256 >> 3) << 17) |
                               (uint32_t(256 >> 4) << 24);

__device__ __forceinline__ void umma_i8_2sm(uint32_t tmem_c, uint64_t da, uint64_t db, uint32_t idesc,
                                            uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, {%5, %6, %7, %8, %9, %10, %11, %12}, p;\n\t}\n" ::"r"(
          tmem_c),
      "l"(da), "l"(db), "r"(idesc), "r"(acc), "r"(0u), "r"(0u), "r"(0u), "r"(0u), "r"(0u), "r"(0u), "r"(0u),
      "r"(0u));
}

__device__ __forceinline__ void umma_commit_2sm(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}

// TMA whose completed bytes are counted on the leader CTA's barrier (peer bit cleared)
__device__ __forceinline__ void tma_load_2d_2sm(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];\n" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar) & 0xFEFFFFFFu), "r"(x), "r"(y)
      : "memory");
}

template <class Epi, int NB>
__global__ void __launch_bounds__(kI8Threads2, 1)
    i8gemm_2sm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int K,
                      int pairs_m, int tiles_n, int group, Epi epi) {
  if (epi.skip()) return;  // uniform over the grid (e.g. an unused Ozaki modulus)
  using Cfg = I8S2<NB>;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(base + size_t(Cfg::kStages) * Cfg::kStageBytes);
  uint64_t* empty = full + Cfg::kStages;
  uint64_t* acc_full = empty + Cfg::kStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_full + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rank = static_cast<int>(cluster_rank());
  const int cl = blockIdx.x >> 1;
  int pm, tn;
  grouped_tile(cl, pairs_m, tiles_n, group, pm, tn);
  const int m0 = pm * 256 + rank * 128;  // this CTA's accumulator rows
  const int n0 = tn * (256 * NB);
  const int KB = K / kI8BK;
  constexpr uint16_t kBoth = 0x3;
  constexpr uint32_t kCols = 256 * NB;

  if (threadIdx.x == 0) {
    for (int s = 0; s < Cfg::kStages; ++s) {
      mbar_init(&full[s], 1);   // leader: its producer's expect_tx (both CTAs' bytes)
      mbar_init(&empty[s], 1);  // the leader's MMA commit
    }
    mbar_init(acc_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(kCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync_all();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tmA) : "memory");
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tmB) : "memory");
      for (int kb = 0; kb < KB; ++kb) {
        const int s = kb % Cfg::kStages;
        if (kb >= Cfg::kStages) mbar_wait(&empty[s], ((kb / Cfg::kStages) - 1) & 1);
        unsigned char* sa = base + size_t(s) * Cfg::kStageBytes;
        if (rank == 0) mbar_expect_tx(&full[s], 2 * Cfg::kStageBytes);
        tma_load_2d_2sm(sa, &tmA, &full[s], kb * kI8BK, m0);
#pragma unroll
        for (int b = 0; b < NB; ++b)
          tma_load_2d_2sm(sa + (1 + b) * 128 * kI8BK, &tmB, &full[s], kb * kI8BK, n0 + b * 256 + rank * 128);
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      for (int kb = 0; kb < KB; ++kb) {
        const int s = kb % Cfg::kStages;
        mbar_wait(&full[s], (kb / Cfg::kStages) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t sa = smem_u32(base + size_t(s) * Cfg::kStageBytes);
        const uint64_t da = umma_desc_sw128(sa);
#pragma unroll
        for (int k = 0; k < kI8BK / 32; ++k)
#pragma unroll
          for (int b = 0; b < NB; ++b)
            umma_i8_2sm(tmem + uint32_t(b * 256), da + 2 * k, umma_desc_sw128(sa + (1 + b) * 128 * kI8BK) + 2 * k,
                        kI8Idesc2, (kb | k) ? 1u : 0u);
        umma_commit_2sm(&empty[s], kBoth);
      }
      umma_commit_2sm(acc_full, kBoth);
    }
  }
  __syncwarp();
  // Epilogue on all 8 warps (the producer and MMA warps included once their loops end):
  // warp w drains TMEM lane quarter w % 4 (its rows), column half w / 4.
  mbar_wait(acc_full, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  {
    const int quarter = warp & 3, half = warp >> 2;
    const int row = m0 + quarter * 32 + lane;
    const uint32_t trow = tmem + (uint32_t(quarter * 32) << 16);
    constexpr int kHalf = int(kCols) / 2;
#pragma unroll 1
    for (int c = half * kHalf; c < (half + 1) * kHalf; c += 32) {
      uint32_t v[32];
      tmem_ld32(trow + uint32_t(c), v);
      epi(row, n0 + c, v);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  cluster_sync_all();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kCols));
}

// `rows` x `k` int8 (K contiguous, pitch ld bytes), TMA boxes of 128 bytes x box_rows rows.
CUtensorMap make_map_i8(const void* base, int64_t k, int64_t rows, int64_t ld, int box_rows);

// Launch C-tile epilogue `epi` over A (M x K) . B (N x K)^T; M % 128, N % 256, K % 128 == 0,
// lda / ldb in bytes.
template <class Epi>
void launch_i8gemm(cudaStream_t s, int64_t M, int64_t N, int64_t K, const int8_t* A, int64_t lda, const int8_t* B,
                   int64_t ldb, const Epi& epi) {
  if (M % kI8BM || N % kI8BN || K % kI8BK || M <= 0 || N <= 0 || K <= 0)
    throw InvalidArgument("i8 gemm: M % 128, N % 256 and K % 128 must be 0");
  static PerDeviceOnce attr;
  attr.run([] {
    IPT_CUDA(cudaFuncSetAttribute(i8gemm_kernel<Epi>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(kI8SmemBytes)));
    IPT_CUDA(cudaFuncSetAttribute(i8gemm_mc_kernel<Epi>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(kI8SmemBytes)));
    IPT_CUDA(cudaFuncSetAttribute(i8gemm_2sm_kernel<Epi, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(I8S2<1>::kSmem)));
    IPT_CUDA(cudaFuncSetAttribute(i8gemm_2sm_kernel<Epi, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(I8S2<2>::kSmem)));
  });
  const int tiles_m = static_cast<int>(M / kI8BM);
  // IPT_I8_GROUP: M tiles (pairs for the 2-SM kernels) per rasterisation group
  const char* genv = std::getenv("IPT_I8_GROUP");
  const int group = genv && std::atoi(genv) > 0 ? std::atoi(genv) : 8;
  const unsigned grid = static_cast<unsigned>(tiles_m * (N / kI8BN));
  // IPT_I8_KERNEL: 2sm (default when M % 256 == 0), mc (B multicast pair), 1sm
  const char* kenv = std::getenv("IPT_I8_KERNEL");
  const std::string kind = kenv ? kenv : (N % 512 == 0 ? "2sm512" : "2sm");
  const bool wide = kind == "2sm512" && N % 512 == 0;
  if ((kind == "2sm" || wide) && tiles_m % 2 == 0) {
    const CUtensorMap ma2 = make_map_i8(A, K, M, lda, 128);
    const CUtensorMap mb2 = make_map_i8(B, K, N, ldb, 128);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(wide ? grid / 2 : grid);
    cfg.blockDim = dim3(kI8Threads2);
    cfg.dynamicSmemBytes = wide ? I8S2<2>::kSmem : I8S2<1>::kSmem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (wide)
      IPT_CUDA(cudaLaunchKernelEx(&cfg, i8gemm_2sm_kernel<Epi, 2>, ma2, mb2, static_cast<int>(K), tiles_m / 2,
                                  static_cast<int>(N / 512), group, epi));
    else
      IPT_CUDA(cudaLaunchKernelEx(&cfg, i8gemm_2sm_kernel<Epi, 1>, ma2, mb2, static_cast<int>(K), tiles_m / 2,
                                  static_cast<int>(N / 256), group, epi));
    IPT_LAUNCH_CHECK();
    count_launch();
    return;
  }
  const bool multicast = tiles_m % 2 == 0 && kind == "mc";
  const CUtensorMap ma = make_map_i8(A, K, M, lda, kI8BM);
  const CUtensorMap mb = make_map_i8(B, K, N, ldb, multicast ? kI8BN / 2 : kI8BN);
  if (multicast) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kI8Threads);
    cfg.dynamicSmemBytes = kI8SmemBytes;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    IPT_CUDA(cudaLaunchKernelEx(&cfg, i8gemm_mc_kernel<Epi>, ma, mb, static_cast<int>(K), tiles_m,
                                static_cast<int>(N / kI8BN), group, epi));
  } else {
    i8gemm_kernel<Epi><<<grid, kI8Threads, kI8SmemBytes, s>>>(ma, mb, static_cast<int>(K), tiles_m,
                                                                   static_cast<int>(N / kI8BN), group, epi);
  }
  IPT_LAUNCH_CHECK();
  count_launch();
}

}  // namespace iptb
