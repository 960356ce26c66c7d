// lora_patch_tc.cu — K1 for bf16 serving weights: TMA-staged, warp-specialised,
// persistent LoRA patch with the rank contraction on tcgen05 (TMEM accumulator).
//
//   W_out[r, c] = bf16( fma(sign*scale, sum_k A[r,k] * B[c,k], float(W_in[r,c])) )
//
// Same arithmetic contract as lora_patch.cu (addonsim/lora.py:84-95: one W
// read-modify-write per element, single rounding, no materialised delta); this
// unit is the B200-native fast path for the whole-UNet patch set.
//
// Data movement (the kernel is HBM-bound: 4 B of W traffic per element vs
// 2R flops, intensity R/2 << the ~256 flop/B ridge):
//   * W moves as 128 x 64 bf16 boxes (16 KB, 128B-swizzled) through a ring of
//     S shared-memory slots: TMA load (cp.async.bulk.tensor) -> epilogue RMW in
//     shared memory -> TMA store.  The ring keeps S*16 KB of W in flight per SM.
//   * Factors are pre-packed once per adapter set (sdb_lora_pack) into the
//     UMMA canonical K-major SWIZZLE_128B layout, so they move with plain bulk
//     copies: the B panel (256 output columns x R, plus the low-part blocks
//     of scale-folded adapters, see the packing section) stays resident while
//     the CTA walks up to 8 row tiles of that panel; the A tile (128 rows x R) is
//     streamed per row tile in 64-deep K blocks through a 2-stage ring
//     (L2-resident: its re-read costs R/256 of the W read).
//   * tcgen05 path: one elected thread issues ceil(R/16) MMAs of
//     M=128 x N=256 x K=16 (kind::f16, bf16 in, fp32 accumulate) into one of
//     two 256-column TMEM accumulators; the 8 epilogue warps read their 32
//     TMEM lanes with tcgen05.ld while the next tile's MMA runs in the other.
// Roles: warps 0-7 epilogue (TMEM lane quadrant x column half), warp 8
// producer (TMA), warp 9 MMA issuer + TMEM allocator.  One CTA per SM, grid-strided over units.
#include <cuda.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "ptx.cuh"
#include "tcgen05.cuh"

namespace sdb {
namespace {

constexpr int kBM = 128;                 // rows per tile (TMEM lanes)
constexpr int kBN = 256;                  // columns per tile / B panel (UMMA N)
constexpr int kBoxN = 64;                 // W box width (128 B of bf16: one swizzle row)
constexpr int kBoxBytes = kBM * kBoxN * 2;          // 16 KB
constexpr int kKB = 64;                   // K elements per packed block (one 128 B row)
constexpr int kABlockBytes = kBM * 128;   // 16 KB per K block of an A tile
constexpr int kBBlockBytes = kBN * 128;   // 32 KB per K block of a B panel
constexpr int kUnitTiles = 8;             // row tiles per work unit (B panel reuse)
constexpr int kEpiWarps = 8;              // 2 warps per TMEM lane quadrant (column halves)
constexpr int kEpiThreads = kEpiWarps * 32;
constexpr int kProducerWarp = kEpiWarps;       // W boxes
constexpr int kMmaWarp = kEpiWarps + 1;
constexpr int kFactorWarp = kEpiWarps + 2;      // B panel + A K-blocks
constexpr int kThreads = (kEpiWarps + 3) * 32;
constexpr int kMaxKB = 4;                 // rank <= 256
constexpr int kAStages = 2;               // A K-blocks in flight
constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kBN >> 3) << 17) |
                            ((uint32_t)(kBM >> 4) << 24);   // f32 accum, bf16 A/B, K-major, 128x256

struct TcJob {
  const uint8_t* a;   // packed A: [m_tiles][kb][128 rows][128 B]
  const uint8_t* b;   // packed B: [n_tiles][bkb][256 rows][128 B]
  int64_t h1, h2;
  int32_t kb, rank;       // A K-blocks (= high-part B K-blocks), stacked rank
  float scale;
  int32_t map_in, map_out;
  int32_t map_a, map_b;   // tensor maps over the packed factors (CTA-pair kernel)
  int32_t mt;             // row tiles of W
  int32_t bkb;            // B-panel K-blocks: kb high parts + the low parts (see lo_of)
  uint32_t lo_of;         // byte a: 0, or 1 + the B-panel block holding the low part A block a also multiplies
  int32_t pad;
};

// The B panel's first kb blocks are the (unscaled or high-part) stacked
// factors; A K-block a also multiplies low-part block lo_block(J, a) when the
// scale-folded sources touch it (hi/lo split, see the packing section)
__device__ __forceinline__ int lo_block(const TcJob& J, int a) {
  return (int)((J.lo_of >> (8 * a)) & 0xFF) - 1;
}
struct TcUnit {
  int32_t job, n_tile, m_begin, m_end;
};

// ---- PTX helpers (mbarriers, bulk copies, L2 policies: ptx.cuh) ------------
// L2 policies: W is streamed exactly once (evict-first); the packed factors are
// re-read by every column panel / row tile (evict-last keeps them resident).
__device__ __forceinline__ float bf16lo(uint32_t u) { return __uint_as_float(u << 16); }
__device__ __forceinline__ float bf16hi(uint32_t u) { return __uint_as_float(u & 0xFFFF0000u); }
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}

// Epilogue update of 32 columns (4 swizzled 16 B chunks) of this thread's row.
__device__ __forceinline__ void rmw32(uint8_t* row, int r, int chunk0, const float (&v)[32], float ss) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    uint4* p = reinterpret_cast<uint4*>(row + (((chunk0 + j) ^ (r & 7)) << 4));
    uint4 w = *p;
    uint32_t* wu = reinterpret_cast<uint32_t*>(&w);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float lo = fmaf(ss, v[8 * j + 2 * e], bf16lo(wu[e]));
      const float hi = fmaf(ss, v[8 * j + 2 * e + 1], bf16hi(wu[e]));
      wu[e] = pack_bf16(lo, hi);
    }
    *p = w;
  }
}

template <int BN>
__global__ void __launch_bounds__(kThreads, 1)
lora_patch_tma_kernel(const CUtensorMap* __restrict__ maps, const TcJob* __restrict__ jobs,
                      const TcUnit* __restrict__ units, int n_units, float sign, int kb_max, int n_slots) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int kPanelBlock = BN * 128;                 // bytes of one K block of the B panel
  constexpr uint32_t kIdescBN = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                                ((uint32_t)(kBM >> 4) << 24);   // f32 accum, bf16 A/B, K-major, 128 x BN
  uint8_t* sB = smem;                                   // kb_max * BN * 128 B: resident B panel
  uint8_t* sA = sB + kb_max * kPanelBlock;              // kAStages * 16 KB: streamed A K-blocks
  uint8_t* sW = sA + kAStages * kABlockBytes;           // n_slots * 16 KB: W box ring
  uint64_t* bars = reinterpret_cast<uint64_t*>(sW + n_slots * kBoxBytes);
  // barrier indices
  const int B_FULL = 0, B_EMPTY = 1, A_FULL = 2, A_EMPTY = A_FULL + kAStages, T_FULL = A_EMPTY + kAStages;
  const int T_EMPTY = T_FULL + 2, W_FULL = T_EMPTY + 2;
  const int W_EMPTY = W_FULL + n_slots;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + W_EMPTY + n_slots);
  auto bar = [&](int i) { return smem_u32(bars + i); };

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    mbar_init(bar(B_FULL), 1);
    mbar_init(bar(B_EMPTY), 1);           // tcgen05.commit after the unit's last MMA
    for (int i = 0; i < kAStages; ++i) {
      mbar_init(bar(A_FULL + i), 1);
      mbar_init(bar(A_EMPTY + i), 1);     // tcgen05.commit after the MMAs reading the stage
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(bar(T_FULL + i), 1);
      mbar_init(bar(T_EMPTY + i), kEpiWarps);
    }
    for (int i = 0; i < n_slots; ++i) {
      mbar_init(bar(W_FULL + i), 1);
      mbar_init(bar(W_EMPTY + i), 4);   // the 4 warps (quadrants) of the owning group
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kMmaWarp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                 "r"(2 * BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  if (warp == kFactorWarp) {
    // ===================== factor producer: B panel, A K-blocks =====================
    // (its own warp: A loads never queue behind a full W ring)
    if (lane == 0) {
      const uint64_t keep = policy_evict_last();
      int b_cnt = 0, a_st = 0, a_round = 0;
      for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
        const TcUnit un = units[u];
        const TcJob& J = jobs[un.job];
        if (b_cnt > 0) mbar_wait(bar(B_EMPTY), (b_cnt - 1) & 1);
        mbar_expect_tx(bar(B_FULL), J.bkb * kPanelBlock);
        if (BN == kBN) {
          bulk_g2s(smem_u32(sB), J.b + (size_t)un.n_tile * J.bkb * kBBlockBytes, J.bkb * kBBlockBytes, bar(B_FULL),
                   keep);
        } else {  // a BN-wide half of a packed 256-wide panel: one copy per K block
          const int p256 = un.n_tile / (kBN / BN), hh = un.n_tile % (kBN / BN);
          for (int kb = 0; kb < J.bkb; ++kb)
            bulk_g2s(smem_u32(sB + kb * kPanelBlock),
                     J.b + (((size_t)p256 * J.bkb + kb) * kBN + (size_t)hh * BN) * 128, kPanelBlock, bar(B_FULL),
                     keep);
        }
        ++b_cnt;
        for (int m = un.m_begin; m < un.m_end; ++m) {
          for (int kb = 0; kb < J.kb; ++kb) {
            if (a_round > 0) mbar_wait(bar(A_EMPTY + a_st), (a_round - 1) & 1);
            mbar_expect_tx(bar(A_FULL + a_st), kABlockBytes);
            bulk_g2s(smem_u32(sA + a_st * kABlockBytes), J.a + ((size_t)m * J.kb + kb) * kABlockBytes, kABlockBytes,
                     bar(A_FULL + a_st), keep);
            if (++a_st == kAStages) { a_st = 0; ++a_round; }
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == kProducerWarp) {
    // ===================== W producer =====================
    if (lane == 0) {
      const uint64_t stream = policy_evict_first();
      int w_slot = 0, w_round = 0;
      for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
        const TcUnit un = units[u];
        const TcJob& J = jobs[un.job];
        const CUtensorMap* min = maps + J.map_in;
        prefetch_map(min);
        const int64_t ncols = std::min<int64_t>(BN, J.h2 - (int64_t)un.n_tile * BN);
        const int nbox = (int)((ncols + kBoxN - 1) / kBoxN);
        for (int m = un.m_begin; m < un.m_end; ++m) {
          for (int bx = 0; bx < nbox; ++bx) {
            if (w_round > 0) mbar_wait(bar(W_EMPTY + w_slot), (w_round - 1) & 1);
            mbar_expect_tx(bar(W_FULL + w_slot), kBoxBytes);
            tma_load_2d(smem_u32(sW + w_slot * kBoxBytes), min, un.n_tile * BN + bx * kBoxN, m * kBM,
                        bar(W_FULL + w_slot), stream);
            if (++w_slot == n_slots) { w_slot = 0; ++w_round; }
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == kMmaWarp) {
    // ===================== MMA issuer (one thread) =====================
    if (lane == 0) {
      int tile = 0, b_cnt = 0, a_cnt = 0;
      for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
        const TcUnit un = units[u];
        const TcJob& J = jobs[un.job];
        const int nks = (J.rank + 15) / 16;     // K steps of 16 (zero-padded)
        mbar_wait(bar(B_FULL), b_cnt & 1);
        for (int m = un.m_begin; m < un.m_end; ++m, ++tile) {
          const int buf = tile & 1;
          if (tile >= 2) mbar_wait(bar(T_EMPTY + buf), ((tile >> 1) - 1) & 1);
          const uint32_t d = tmem_base + buf * BN;
          for (int kb = 0; kb < J.kb; ++kb, ++a_cnt) {
            const int st = a_cnt & (kAStages - 1);
            mbar_wait(bar(A_FULL + st), (a_cnt / kAStages) & 1);
            tc_fence_after();
            const int ks_end = std::min(4, nks - kb * 4);
            const int lb = lo_block(J, kb);
            for (int ks = 0; ks < ks_end; ++ks) {
              const uint64_t ad = sw128_desc(smem_u32(sA + st * kABlockBytes + ks * 32));
              tc_mma(d, ad, sw128_desc(smem_u32(sB + kb * kPanelBlock + ks * 32)), kIdescBN, (kb | ks) ? 1u : 0u);
              if (lb >= 0) tc_mma(d, ad, sw128_desc(smem_u32(sB + lb * kPanelBlock + ks * 32)), kIdescBN, 1u);
            }
            tc_commit(bar(A_EMPTY + st));       // stage free once these MMAs completed
          }
          tc_commit(bar(T_FULL + buf));          // accumulator complete
        }
        tc_commit(bar(B_EMPTY));
        ++b_cnt;
      }
    }
    __syncwarp();
  } else {
    // ===================== epilogue (warps 0-7) =====================
    // warp e owns TMEM lane quadrant q = e & 3 (rows 32q..32q+31) and, with
    // the other 3 warps of its group g = e >> 2, every other W box: no
    // cross-warp barrier — each warp TMA-stores its own 32-row sub-box.
    const int q = warp & 3, grp = warp >> 2;
    const int r = (q << 5) | lane;             // tile row == TMEM lane
    int box = 0;                               // running box counter (group ownership)
    int tile = 0, w_slot = 0, w_round = 0;
    int pending = -1;                          // slot whose TMA store may still be reading smem
    const uint64_t stream = policy_evict_first();
    for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
      const TcUnit un = units[u];
      const TcJob& J = jobs[un.job];
      const CUtensorMap* mout = maps + J.map_out;
      const float ss = sign * J.scale;
      const int64_t ncols = std::min<int64_t>(BN, J.h2 - (int64_t)un.n_tile * BN);
      const int nbox = (int)((ncols + kBoxN - 1) / kBoxN);
      for (int m = un.m_begin; m < un.m_end; ++m, ++tile) {
        const int buf = tile & 1;
        mbar_wait(bar(T_FULL + buf), (tile >> 1) & 1);
        tc_fence_after();
        for (int bx = 0; bx < nbox; ++bx) {
          const int slot = w_slot, round = w_round;
          if (++w_slot == n_slots) { w_slot = 0; ++w_round; }
          const bool mine = ((box++ & 1) == grp);   // warp-uniform
          if (!mine) continue;
          mbar_wait(bar(W_FULL + slot), round & 1);
          uint8_t* row = sW + slot * kBoxBytes + r * 128;
#pragma unroll
          for (int hf = 0; hf < 2; ++hf) {
            float v[32];
            tc_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + buf * BN + bx * kBoxN + hf * 32, v);
            rmw32(row, r, hf * 4, v, ss);
          }
          fence_proxy_async();
          __syncwarp();
          if (lane == 0) {
            // this warp's 32 rows of the box; keep one store in flight and
            // release the PREVIOUS slot once its smem read is done
            tma_store_2d(mout, un.n_tile * BN + bx * kBoxN, m * kBM + q * 32,
                         smem_u32(sW + slot * kBoxBytes + q * 32 * 128), stream);
            if (pending >= 0) {
              tma_store_wait_read1();
              mbar_arrive(bar(W_EMPTY + pending));
            }
            pending = slot;
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(bar(T_EMPTY + buf));
      }
    }
    if (lane == 0) {
      if (pending >= 0) {
        tma_store_wait_read();
        mbar_arrive(bar(W_EMPTY + pending));
      }
      tma_store_wait_all();
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(2 * BN));
  }
}

// ---- CTA-pair variant (cta_group::2) ------------------------------------------
// The B panel is what limits the W ring at high rank: 256 columns x R bf16 is
// 128 KB at R = 256, leaving 4 W slots.  A pair of CTAs on one TPC shares it:
// tcgen05.mma.cta_group::2 computes M = 256 rows (128 per CTA, each CTA's A
// tile in its own smem) x N = 256 columns, with B split along N — each CTA
// holds only its half of the panel (64 KB at R = 256), so both keep an 8-slot
// W ring.  Each CTA's TMEM receives its own 128 rows x 256 columns, so the
// epilogue and the W traffic are unchanged.  The leader (rank 0) issues the
// MMAs; factor loads of both CTAs complete on the leader's barriers
// (cp.async.bulk.tensor .cta_group::2) and the MMA commits multicast to both.
// (cluster / CTA-pair helpers: tcgen05.cuh)
constexpr int kPairUnitTiles = 16;   // row tiles per pair unit (8 per CTA: same B reuse)
constexpr int kHalfBlock = 128 * 128; // one K block of half a B panel (128 columns x 64 K)
constexpr int kMaxSlots = 10;

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
lora_patch_pair_kernel(const CUtensorMap* __restrict__ maps, const TcJob* __restrict__ jobs,
                       const TcUnit* __restrict__ units, int n_units, float sign, int kb_max, int n_slots,
                       int na) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr uint32_t kIdesc2 = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kBN >> 3) << 17) |
                               ((uint32_t)(256 >> 4) << 24);   // f32 accum, bf16, K-major, M256 x N256
  uint8_t* sB = smem;                                   // kb_max x 16 KB: this CTA's half of the B panel
  uint8_t* sA = sB + kb_max * kHalfBlock;               // na x 16 KB: streamed A K-blocks
  uint8_t* sW = sA + na * kABlockBytes;                 // n_slots x 16 KB
  uint64_t* bars = reinterpret_cast<uint64_t*>(sW + n_slots * kBoxBytes);
  const int B_FULL = 0, B_EMPTY = 1, A_FULL = 2, A_EMPTY = A_FULL + na, T_FULL = A_EMPTY + na;
  const int T_EMPTY = T_FULL + 2, W_FULL = T_EMPTY + 2;
  const int W_EMPTY = W_FULL + n_slots;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + W_EMPTY + n_slots);
  auto bar = [&](int i) { return smem_u32(bars + i); };

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t cta = cluster_ctarank();
  const bool leader = cta == 0;
  const int cid = (int)cluster_idx(), ncl = (int)cluster_count();

  if (threadIdx.x == 0) {
    mbar_init(bar(B_FULL), 1);
    mbar_init(bar(B_EMPTY), 1);
    for (int i = 0; i < na; ++i) {
      mbar_init(bar(A_FULL + i), 1);
      mbar_init(bar(A_EMPTY + i), 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(bar(T_FULL + i), 1);
      mbar_init(bar(T_EMPTY + i), 2 * kEpiWarps);   // both CTAs' epilogue warps
    }
    for (int i = 0; i < n_slots; ++i) {
      mbar_init(bar(W_FULL + i), 1);
      mbar_init(bar(W_EMPTY + i), 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kMmaWarp) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                 "r"(2 * kBN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  if (warp == kFactorWarp) {
    // factor producer: this CTA's half of the B panel and its A K-blocks,
    // completing on the leader's barriers
    if (lane == 0) {
      const uint64_t keep = policy_evict_last();
      int b_cnt = 0, a_st = 0, a_round = 0;
      for (int u = cid; u < n_units; u += ncl) {
        const TcUnit un = units[u];
        const TcJob& J = jobs[un.job];
        const CUtensorMap* ma = maps + J.map_a;
        const CUtensorMap* mb = maps + J.map_b;
        if (b_cnt > 0) mbar_wait(bar(B_EMPTY), (b_cnt - 1) & 1);
        if (leader) mbar_expect_tx(bar(B_FULL), 2 * J.bkb * kHalfBlock);
        for (int kb = 0; kb < J.bkb; ++kb)
          tma_load_2d_pair(smem_u32(sB + kb * kHalfBlock), mb, 0, (un.n_tile * J.bkb + kb) * kBN + (int)cta * 128,
                           mapa_shared(bar(B_FULL), 0), keep);
        ++b_cnt;
        for (int m0 = un.m_begin; m0 < un.m_end; m0 += 2) {
          // past the last row tile the follower multiplies a valid (ignored) A tile
          const int mload = std::min(m0 + (int)cta, J.mt - 1);
          for (int kb = 0; kb < J.kb; ++kb) {
            if (a_round > 0) mbar_wait(bar(A_EMPTY + a_st), (a_round - 1) & 1);
            if (leader) mbar_expect_tx(bar(A_FULL + a_st), 2 * kABlockBytes);
            tma_load_2d_pair(smem_u32(sA + a_st * kABlockBytes), ma, 0, (mload * J.kb + kb) * kBM,
                             mapa_shared(bar(A_FULL + a_st), 0), keep);
            if (++a_st == na) { a_st = 0; ++a_round; }
          }
        }
      }
      // drain: the leader's last multicast commits must land before this CTA exits
      for (int s = 0; s < na; ++s) {
        const int uses = a_round + (s < a_st ? 1 : 0);
        if (uses > 0) mbar_wait(bar(A_EMPTY + s), (uses - 1) & 1);
      }
      if (b_cnt > 0) mbar_wait(bar(B_EMPTY), (b_cnt - 1) & 1);
    }
    __syncwarp();
  } else if (warp == kProducerWarp) {
    // W producer: this CTA's row tiles only
    if (lane == 0) {
      const uint64_t stream = policy_evict_first();
      int w_slot = 0, w_round = 0;
      for (int u = cid; u < n_units; u += ncl) {
        const TcUnit un = units[u];
        const TcJob& J = jobs[un.job];
        const CUtensorMap* min = maps + J.map_in;
        prefetch_map(min);
        const int64_t ncols = std::min<int64_t>(kBN, J.h2 - (int64_t)un.n_tile * kBN);
        const int nbox = (int)((ncols + kBoxN - 1) / kBoxN);
        for (int m = un.m_begin + (int)cta; m < un.m_end; m += 2) {
          for (int bx = 0; bx < nbox; ++bx) {
            if (w_round > 0) mbar_wait(bar(W_EMPTY + w_slot), (w_round - 1) & 1);
            mbar_expect_tx(bar(W_FULL + w_slot), kBoxBytes);
            tma_load_2d(smem_u32(sW + w_slot * kBoxBytes), min, un.n_tile * kBN + bx * kBoxN, m * kBM,
                        bar(W_FULL + w_slot), stream);
            if (++w_slot == n_slots) { w_slot = 0; ++w_round; }
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == kMmaWarp) {
    if (leader && lane == 0) {
      int tile = 0, b_cnt = 0, a_st = 0, a_round = 0;
      for (int u = cid; u < n_units; u += ncl) {
        const TcUnit un = units[u];
        const TcJob& J = jobs[un.job];
        const int nks = (J.rank + 15) / 16;
        mbar_wait(bar(B_FULL), b_cnt & 1);
        for (int m0 = un.m_begin; m0 < un.m_end; m0 += 2, ++tile) {
          const int buf = tile & 1;
          if (tile >= 2) mbar_wait(bar(T_EMPTY + buf), ((tile >> 1) - 1) & 1);
          tc_fence_after();
          const uint32_t d = tmem_base + buf * kBN;
          for (int kb = 0; kb < J.kb; ++kb) {
            const int st = a_st;
            mbar_wait(bar(A_FULL + st), a_round & 1);
            if (++a_st == na) { a_st = 0; ++a_round; }
            tc_fence_after();
            const int ks_end = std::min(4, nks - kb * 4);
            const int lb = lo_block(J, kb);
            for (int ks = 0; ks < ks_end; ++ks) {
              const uint64_t ad = sw128_desc(smem_u32(sA + st * kABlockBytes + ks * 32));
              tc_mma2(d, ad, sw128_desc(smem_u32(sB + kb * kHalfBlock + ks * 32)), kIdesc2, (kb | ks) ? 1u : 0u);
              if (lb >= 0) tc_mma2(d, ad, sw128_desc(smem_u32(sB + lb * kHalfBlock + ks * 32)), kIdesc2, 1u);
            }
            tc_commit2(bar(A_EMPTY + st));
          }
          tc_commit2(bar(T_FULL + buf));
        }
        tc_commit2(bar(B_EMPTY));
        ++b_cnt;
      }
    }
    __syncwarp();
  } else {
    // epilogue: as in the single-CTA kernel, on this CTA's 128 rows
    const int q = warp & 3, grp = warp >> 2;
    const int r = (q << 5) | lane;
    int box = 0, tile = 0, w_slot = 0, w_round = 0, pending = -1;
    const uint64_t stream = policy_evict_first();
    for (int u = cid; u < n_units; u += ncl) {
      const TcUnit un = units[u];
      const TcJob& J = jobs[un.job];
      const CUtensorMap* mout = maps + J.map_out;
      const float ss = sign * J.scale;
      const int64_t ncols = std::min<int64_t>(kBN, J.h2 - (int64_t)un.n_tile * kBN);
      const int nbox = (int)((ncols + kBoxN - 1) / kBoxN);
      for (int m0 = un.m_begin; m0 < un.m_end; m0 += 2, ++tile) {
        const int m = m0 + (int)cta;
        const int buf = tile & 1;
        mbar_wait(bar(T_FULL + buf), (tile >> 1) & 1);
        tc_fence_after();
        if (m < un.m_end) {
          for (int bx = 0; bx < nbox; ++bx) {
            const int slot = w_slot, round = w_round;
            if (++w_slot == n_slots) { w_slot = 0; ++w_round; }
            const bool mine = ((box++ & 1) == grp);
            if (!mine) continue;
            mbar_wait(bar(W_FULL + slot), round & 1);
            uint8_t* row = sW + slot * kBoxBytes + r * 128;
#pragma unroll
            for (int hf = 0; hf < 2; ++hf) {
              float v[32];
              tc_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + buf * kBN + bx * kBoxN + hf * 32, v);
              rmw32(row, r, hf * 4, v, ss);
            }
            fence_proxy_async();
            __syncwarp();
            if (lane == 0) {
              tma_store_2d(mout, un.n_tile * kBN + bx * kBoxN, m * kBM + q * 32,
                           smem_u32(sW + slot * kBoxBytes + q * 32 * 128), stream);
              if (pending >= 0) {
                tma_store_wait_read1();
                mbar_arrive(bar(W_EMPTY + pending));
              }
              pending = slot;
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (leader) mbar_arrive(bar(T_EMPTY + buf));
          else mbar_arrive_remote(mapa_shared(bar(T_EMPTY + buf), 0));
        }
      }
    }
    if (lane == 0) {
      if (pending >= 0) {
        tma_store_wait_read();
        mbar_arrive(bar(W_EMPTY + pending));
      }
      tma_store_wait_all();
    }
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == kMmaWarp) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(2 * kBN));
  }
}

// ---- packing ----------------------------------------------------------------
// Multi-source packing: the stacked adapter set (lora.py:147-160: down' =
// [d_1*f32(s_1) | d_2*f32(s_2) ...], up' = [u_1; u_2 ...]) is assembled while
// packing, straight from each adapter's own factor buffers — no stacked copy.
//
// Exact scales.  Folding s_k into a bf16 A operand would round s_k*d a second
// time (2^-9 relative per factor element) — where W + delta nearly cancels
// that is many bf16 ulps of the result.  Instead the scale carried by the
// largest share of the stacked rank (s_e) is applied in the fp32 epilogue and
// its sources are packed unscaled (exact); for every other source the ratio
// goes into its `up` rows — the B panel, which stays resident in shared
// memory while the CTA walks its row tiles — as x = f32(u) * f32(s_k / s_e)
// split into hi = bf16(x) (in the stacked K-blocks) and lo = bf16(x - hi) (in
// an extra B K-block that the SAME A K-block also multiplies, see lo_block):
// hi + lo carries x to 2^-17 relative, A (down, re-read per column panel) is
// packed once, unscaled.  Only K-blocks that hold a folded source get a low
// block, so equal scales (the serving case: every adapter at one strength)
// cost nothing extra.
constexpr int kMaxSrc = 8;
struct PackSrcs {
  const __nv_bfloat16* down[kMaxSrc];
  const __nv_bfloat16* up[kMaxSrc];
  int64_t ldd[kMaxSrc], ldu[kMaxSrc];
  int koff[kMaxSrc + 1];   // prefix sums of the ranks
  float fold[kMaxSrc];     // s_k / s_e (exactly 1 for the epilogue-scaled sources)
  int n;
  int kb;                  // stacked K-blocks (high parts)
  uint32_t lo_b;           // byte i: the K-block whose low part is B-panel block kb + i
};

struct MultiLayout {
  float epi_scale;
  float fold[kMaxSrc];
  int rank, kb, nlo;
  uint32_t lo_mask, lo_b;
};

int multi_layout(const sdb_lora_src* srcs, int n, MultiLayout* L) {
  if (n < 1 || n > kMaxSrc || !srcs) return fail(SDB_EINVAL, "lora_pack_multi: 1..8 sources");
  L->rank = 0;
  for (int i = 0; i < n; ++i) {
    if (srcs[i].rank < 1) return fail(SDB_EINVAL, "lora_pack_multi: source " + std::to_string(i) + ": bad rank");
    L->rank += srcs[i].rank;
  }
  if (L->rank > kMaxKB * kKB) return fail(SDB_EINVAL, "lora_pack_multi: stacked rank must be <= 256");
  // epilogue scale: the nonzero scale with the largest total rank (first on ties)
  float best = 0.f;
  int best_r = 0;
  for (int i = 0; i < n; ++i) {
    if (srcs[i].scale == 0.f) continue;
    int r = 0;
    for (int j = 0; j < n; ++j)
      if (srcs[j].scale == srcs[i].scale) r += srcs[j].rank;
    if (r > best_r) { best_r = r; best = srcs[i].scale; }
  }
  L->epi_scale = best;
  L->kb = (L->rank + kKB - 1) / kKB;
  L->lo_mask = 0;
  int k0 = 0;
  for (int i = 0; i < n; ++i) {
    L->fold[i] = best == 0.f ? 1.f : srcs[i].scale / best;
    if (L->fold[i] != 1.f)
      for (int b = k0 / kKB; b <= (k0 + srcs[i].rank - 1) / kKB; ++b) L->lo_mask |= 1u << b;
    k0 += srcs[i].rank;
  }
  L->nlo = 0;
  L->lo_b = 0;
  for (int b = 0; b < L->kb; ++b)
    if (L->lo_mask >> b & 1u) L->lo_b |= (uint32_t)b << (8 * L->nlo++);
  return SDB_OK;
}

__device__ __forceinline__ int src_of(const PackSrcs& s, int k) {
  int i = 0;
  while (i + 1 < s.n && k >= s.koff[i + 1]) ++i;
  return i;
}

__global__ void pack_a_multi_kernel(PackSrcs s, int64_t h1, int kbt, int64_t mt, uint4* __restrict__ out) {
  const int rank = s.koff[s.n];
  const int64_t total = mt * kbt * kBM * 8;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i & 7);
    const int64_t rowi = i >> 3;                // (m*kbt + kb)*128 + r
    const int r = (int)(rowi % kBM);
    const int64_t mk = rowi / kBM;
    const int kb = (int)(mk % kbt);
    const int64_t m = mk / kbt;
    const int64_t row = m * kBM + r;
    const int k0 = kb * kKB + c * 8;
    __align__(16) __nv_bfloat16 v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int k = k0 + e;
      v[e] = __float2bfloat16_rn(0.f);
      if (row < h1 && k < rank) {
        const int si = src_of(s, k);
        v[e] = s.down[si][row * s.ldd[si] + (k - s.koff[si])];   // unscaled: the scales live in B / the epilogue
      }
    }
    out[rowi * 8 + (c ^ (r & 7))] = *reinterpret_cast<uint4*>(v);
  }
}

// B: [nt][bkb][256][8 chunks x 16 B]; blocks kb.. hold the low parts
__global__ void pack_b_multi_kernel(PackSrcs s, int64_t h2, int bkb, int64_t nt, uint4* __restrict__ out) {
  const int rank = s.koff[s.n];
  const int64_t total = nt * bkb * 8 * kBN;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int n = (int)(i % kBN);               // fastest: coalesced reads of up rows
    const int64_t q = i / kBN;
    const int c = (int)(q & 7);
    const int64_t nk = q >> 3;                  // nt*bkb + b
    const int b = (int)(nk % bkb);
    const int64_t ntile = nk / bkb;
    const int64_t col = ntile * kBN + n;
    const bool low = b >= s.kb;
    const int kb = low ? (int)((s.lo_b >> (8 * (b - s.kb))) & 0xFF) : b;
    const int k0 = kb * kKB + c * 8;
    __align__(16) __nv_bfloat16 v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int k = k0 + e;
      float x = 0.f;
      if (col < h2 && k < rank) {
        const int si = src_of(s, k);
        x = __bfloat162float(s.up[si][(int64_t)(k - s.koff[si]) * s.ldu[si] + col]) * s.fold[si];
        if (low) x -= __bfloat162float(__float2bfloat16_rn(x));   // exactly 0 for fold == 1
      }
      v[e] = __float2bfloat16_rn(x);
    }
    out[(nk * kBN + n) * 8 + (c ^ (n & 7))] = *reinterpret_cast<uint4*>(v);
  }
}

// A: [mt][kb][128][8 chunks x 16 B], chunk c of row r stored at c ^ (r & 7)
__global__ void pack_a_kernel(const __nv_bfloat16* __restrict__ down, int64_t ldd, int64_t h1, int rank,
                              int kbt, int64_t mt, uint4* __restrict__ out) {
  const int64_t total = mt * kbt * kBM * 8;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i & 7);
    const int64_t rowi = i >> 3;                // (m*kbt + kb)*128 + r
    const int r = (int)(rowi % kBM);
    const int64_t mk = rowi / kBM;
    const int kb = (int)(mk % kbt);
    const int64_t m = mk / kbt;
    const int64_t row = m * kBM + r;
    const int k0 = kb * kKB + c * 8;
    __align__(16) __nv_bfloat16 v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e)
      v[e] = (row < h1 && k0 + e < rank) ? down[row * ldd + k0 + e] : __float2bfloat16_rn(0.f);
    out[rowi * 8 + (c ^ (r & 7))] = *reinterpret_cast<uint4*>(v);
  }
}
// B: [nt][kb][256][8 chunks x 16 B] holding up^T (row n = output column n)
__global__ void pack_b_kernel(const __nv_bfloat16* __restrict__ up, int64_t ldu, int64_t h2, int rank, int kbt,
                              int64_t nt, uint4* __restrict__ out) {
  const int64_t total = nt * kbt * 8 * kBN;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int n = (int)(i % kBN);               // fastest: coalesced reads of up rows
    const int64_t q = i / kBN;
    const int c = (int)(q & 7);
    const int64_t nk = q >> 3;                  // nt*kbt + kb
    const int kb = (int)(nk % kbt);
    const int64_t ntile = nk / kbt;
    const int64_t col = ntile * kBN + n;
    const int k0 = kb * kKB + c * 8;
    __align__(16) __nv_bfloat16 v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e)
      v[e] = (col < h2 && k0 + e < rank) ? up[(int64_t)(k0 + e) * ldu + col] : __float2bfloat16_rn(0.f);
    out[(nk * kBN + n) * 8 + (c ^ (n & 7))] = *reinterpret_cast<uint4*>(v);
  }
}

// ---- host side ----------------------------------------------------------------
int make_w_map(CUtensorMap* map, void* ptr, int64_t h1, int64_t h2, int64_t ldw, int box_rows) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) return fail(SDB_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)h2, (cuuint64_t)h1};
  cuuint64_t strides[1] = {(cuuint64_t)ldw * 2};
  cuuint32_t box[2] = {(cuuint32_t)kBoxN, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, ptr, dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(SDB_EINVAL, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return SDB_OK;
}


// packed factors viewed as rows of 128 B (64 bf16); box = one 128-row K block,
// copied verbatim (the data is already in the SWIZZLE_128B pattern)
int make_f_map(CUtensorMap* map, const void* ptr, int64_t rows) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) return fail(SDB_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)kKB, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)kKB * 2};
  cuuint32_t box[2] = {(cuuint32_t)kKB, (cuuint32_t)kBM};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(SDB_EINVAL, "cuTensorMapEncodeTiled (factors) failed (" + std::to_string((int)r) + ")");
  return SDB_OK;
}
}  // namespace

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
    else
      cudaGetLastError();
  }
  return fn;
}

int tc_kb(int rank) { return (rank + kKB - 1) / kKB; }

void tc_pack_bytes(int64_t h1, int64_t h2, int rank, size_t* a_bytes, size_t* b_bytes) {
  const int64_t kbt = tc_kb(rank);
  *a_bytes = (size_t)((h1 + kBM - 1) / kBM) * kbt * kABlockBytes;
  *b_bytes = (size_t)((h2 + kBN - 1) / kBN) * kbt * kBBlockBytes;
}

int tc_pack(const void* down, int64_t ldd, const void* up, int64_t ldu, int64_t h1, int64_t h2, int rank,
            void* a_out, void* b_out, cudaStream_t st) {
  if (rank < 1 || rank > kMaxKB * kKB) return fail(SDB_EINVAL, "lora_pack: rank must be in [1, 256]");
  if (((uintptr_t)a_out | (uintptr_t)b_out) & 1023) return fail(SDB_EINVAL, "lora_pack: outputs must be 1024-B aligned");
  const int kbt = tc_kb(rank);
  const int64_t mt = (h1 + kBM - 1) / kBM, nt = (h2 + kBN - 1) / kBN;
  const int64_t na = mt * kbt * kBM * 8, nb = nt * kbt * 8 * kBN;
  pack_a_kernel<<<(unsigned)std::min<int64_t>((na + 255) / 256, 65535), 256, 0, st>>>(
      static_cast<const __nv_bfloat16*>(down), ldd, h1, rank, kbt, mt, static_cast<uint4*>(a_out));
  if (int rc = check_launch("pack_a_kernel")) return rc;
  pack_b_kernel<<<(unsigned)std::min<int64_t>((nb + 255) / 256, 65535), 256, 0, st>>>(
      static_cast<const __nv_bfloat16*>(up), ldu, h2, rank, kbt, nt, static_cast<uint4*>(b_out));
  return check_launch("pack_b_kernel");
}

int tc_pack_multi_layout(const sdb_lora_src* srcs, int n_src, int64_t h1, int64_t h2, size_t* a_bytes,
                         size_t* b_bytes, float* epi_scale, int32_t* lo_mask) {
  MultiLayout L;
  if (int rc = multi_layout(srcs, n_src, &L)) return rc;
  if (a_bytes) *a_bytes = (size_t)((h1 + kBM - 1) / kBM) * L.kb * kABlockBytes;
  if (b_bytes) *b_bytes = (size_t)((h2 + kBN - 1) / kBN) * (L.kb + L.nlo) * kBBlockBytes;
  if (epi_scale) *epi_scale = L.epi_scale;
  if (lo_mask) *lo_mask = (int32_t)L.lo_mask;
  return SDB_OK;
}

int tc_pack_multi(const sdb_lora_src* srcs, int n_src, int64_t h1, int64_t h2, void* a_out, void* b_out,
                  cudaStream_t st) {
  MultiLayout L;
  if (int rc = multi_layout(srcs, n_src, &L)) return rc;
  if (((uintptr_t)a_out | (uintptr_t)b_out) & 1023)
    return fail(SDB_EINVAL, "lora_pack_multi: outputs must be 1024-B aligned");
  PackSrcs s;
  std::memset(&s, 0, sizeof(s));
  s.n = n_src;
  s.koff[0] = 0;
  for (int i = 0; i < n_src; ++i) {
    if (!srcs[i].down || !srcs[i].up || srcs[i].ldd < srcs[i].rank || srcs[i].ldu < h2)
      return fail(SDB_EINVAL, "lora_pack_multi: source " + std::to_string(i) + ": bad pointer / stride");
    s.down[i] = static_cast<const __nv_bfloat16*>(srcs[i].down);
    s.up[i] = static_cast<const __nv_bfloat16*>(srcs[i].up);
    s.ldd[i] = srcs[i].ldd;
    s.ldu[i] = srcs[i].ldu;
    s.fold[i] = L.fold[i];
    s.koff[i + 1] = s.koff[i] + srcs[i].rank;
  }
  s.kb = L.kb;
  s.lo_b = L.lo_b;
  const int bkb = L.kb + L.nlo;
  const int64_t mt = (h1 + kBM - 1) / kBM, nt = (h2 + kBN - 1) / kBN;
  const int64_t na = mt * L.kb * kBM * 8, nb = nt * bkb * 8 * kBN;
  pack_a_multi_kernel<<<(unsigned)std::min<int64_t>((na + 255) / 256, 65535), 256, 0, st>>>(
      s, h1, L.kb, mt, static_cast<uint4*>(a_out));
  if (int rc = check_launch("pack_a_multi_kernel")) return rc;
  pack_b_multi_kernel<<<(unsigned)std::min<int64_t>((nb + 255) / 256, 65535), 256, 0, st>>>(
      s, h2, bkb, nt, static_cast<uint4*>(b_out));
  return check_launch("pack_b_multi_kernel");
}

// Kernel choice.  The B panel (256 x Rpad bf16) stays resident in shared
// memory.  The single-CTA kernel holds all of it (64 KB at rank 128, 128 KB
// at 256, which squeezes the W ring to 4 slots); the CTA-pair kernel splits
// it across the two CTAs of a TPC, keeping 8-10 W slots at every rank.  The
// pair kernel measured faster at every rank (round 1, SDXL all 794 matrices:
// R=8 1.91 vs 2.04 ms, R=128 2.00 vs 2.20, R=232 2.43 vs 3.61), so auto = pair;
// sdb_lora_tc_set_mode forces one kernel (tests, probes).  The chosen kernel
// is folded into the plan's opaque kb_max word (kb | mode << 8) so a plan
// always launches the kernel it was built for.
static int g_tc_mode = 0;   // 0 auto, 1 single CTA, 2 CTA pair
static int pick_mode(int kb_max) {
  if (g_tc_mode == 1 || g_tc_mode == 2) return g_tc_mode;
  // one 64-wide K block (stacked rank <= 64): the B panel is 32 KB, the
  // single-CTA kernel keeps a deep W ring on its own and, with the balanced
  // unit order, measured 1.88 ms vs the pair's 1.91 (all SDXL matrices, r64)
  return kb_max <= 1 ? 1 : 2;
}

// Blob layout: [maps: 4*n_jobs CUtensorMap (64 B aligned)] [jobs] [units]
// maps per job: W in (128-row load boxes), W out (32-row store boxes),
// packed A, packed B (128-row K blocks; CTA-pair kernel).
int tc_plan(const sdb_lora_tc_job* jobs, int n_jobs, void* blob, size_t blob_bytes, size_t* needed, int* n_units_out,
            int* kb_max_out) {
  if (n_jobs <= 0 || !jobs) return fail(SDB_EINVAL, "lora_tc_plan: no jobs");
  std::vector<TcUnit> units;
  int kb_max = 1, bkb_max = 1;   // A K-blocks, B-panel K-blocks (incl. low parts)
  for (int j = 0; j < n_jobs; ++j) {
    const sdb_lora_tc_job& J = jobs[j];
    if (J.h1 <= 0 || J.h2 <= 0 || J.rank < 1 || J.rank > kMaxKB * kKB)
      return fail(SDB_EINVAL, "lora_tc_plan: job " + std::to_string(j) + ": bad shape or rank (1..256)");
    if ((uint32_t)J.lo_mask >> tc_kb(J.rank))
      return fail(SDB_EINVAL, "lora_tc_plan: job " + std::to_string(j) + ": lo_mask names a K block past the rank");
    bkb_max = std::max(bkb_max, tc_kb(J.rank) + __builtin_popcount((uint32_t)J.lo_mask));
    if (J.ldw % 8 != 0 || ((uintptr_t)J.w_in & 15) || ((uintptr_t)J.w_out & 15))
      return fail(SDB_EINVAL, "lora_tc_plan: job " + std::to_string(j) + ": W rows must be 16-B aligned (ldw % 8 == 0)");
    if (((uintptr_t)J.a_packed | (uintptr_t)J.b_packed) & 1023)
      return fail(SDB_EINVAL, "lora_tc_plan: job " + std::to_string(j) + ": packed factors must be 1024-B aligned");
    kb_max = std::max(kb_max, tc_kb(J.rank));
  }
  const int mode = pick_mode(kb_max);
  const int unit_tiles = mode == 2 ? kPairUnitTiles : kUnitTiles;
  for (int j = 0; j < n_jobs; ++j) {
    const sdb_lora_tc_job& J = jobs[j];
    const int64_t mt = (J.h1 + kBM - 1) / kBM, nt = (J.h2 + kBN - 1) / kBN;
    for (int64_t n = 0; n < nt; ++n)
      for (int64_t m = 0; m < mt; m += unit_tiles)
        units.push_back({j, (int32_t)n, (int32_t)m, (int32_t)std::min<int64_t>(mt, m + unit_tiles)});
  }
  // Static balance: the kernel hands unit u to CTA (pair) u % ncl.  Units
  // range from 1 to unit_tiles row tiles (a 320-row matrix is one 3-tile
  // unit), so plain job order leaves some CTAs ~7% more work than others
  // (ncu: SM active 93% of the elapsed cycles); sort by size and deal the
  // units out boustrophedon (round k forward for even k, backward for odd
  // k) so every CTA's total is near the mean.  Single-CTA kernel: largest
  // first (r64: 2.06 -> 1.88 ms, R=232: 3.60 -> 2.90 ms).  CTA pair: smallest
  // first — a 1-tile unit idles half the pair, and dealing those last left
  // every pair half-idle at the tail (largest-first was 2% slower at
  // R=128); smallest-first is neutral at R <= 128 and 0.5% faster at R=232.
  // SDB_K1_BALANCE=0 keeps job order (probe knob).
  static int balance = -1;
  if (balance < 0) {
    const char* e = getenv("SDB_K1_BALANCE");
    balance = e ? atoi(e) : 1;
  }
  if (balance) {
    const int ncl = mode == 2 ? kNumSMs / 2 : kNumSMs;
    auto elems = [&](const TcUnit& u) {          // W elements the unit reads and writes
      const sdb_lora_tc_job& J = jobs[u.job];
      const int64_t rows = std::min<int64_t>(J.h1, (int64_t)u.m_end * kBM) - (int64_t)u.m_begin * kBM;
      const int64_t cols = std::min<int64_t>(J.h2 - (int64_t)u.n_tile * kBN, kBN);
      return rows * cols;
    };
    std::vector<TcUnit> sorted(units);
    if (mode == 2)
      std::stable_sort(sorted.begin(), sorted.end(),
                       [&](const TcUnit& a, const TcUnit& b) { return elems(a) < elems(b); });
    else
      std::stable_sort(sorted.begin(), sorted.end(),
                       [&](const TcUnit& a, const TcUnit& b) { return elems(a) > elems(b); });
    for (size_t k = 0; k * ncl < sorted.size(); ++k) {
      const size_t b = k * ncl, e = std::min(sorted.size(), b + ncl);
      if (k & 1) std::reverse(sorted.begin() + b, sorted.begin() + e);
    }
    units.swap(sorted);
  }
  const size_t maps_b = (size_t)4 * n_jobs * sizeof(CUtensorMap);
  const size_t jobs_b = (size_t)n_jobs * sizeof(TcJob);
  const size_t units_b = units.size() * sizeof(TcUnit);
  const size_t need = maps_b + jobs_b + units_b;
  if (needed) *needed = need;
  if (n_units_out) *n_units_out = (int)units.size();
  if (kb_max_out) *kb_max_out = bkb_max | (mode << 8) | (kb_max << 12);
  if (!blob) return SDB_OK;
  if (blob_bytes < need) return fail(SDB_EINVAL, "lora_tc_plan: blob too small");
  uint8_t* base = static_cast<uint8_t*>(blob);
  CUtensorMap* maps = reinterpret_cast<CUtensorMap*>(base);
  TcJob* tj = reinterpret_cast<TcJob*>(base + maps_b);
  for (int j = 0; j < n_jobs; ++j) {
    const sdb_lora_tc_job& J = jobs[j];
    const int kb = tc_kb(J.rank);
    int nlo = 0;
    uint32_t lo_of = 0;     // byte a: 1 + the B-panel block of A block a's low part
    for (int b = 0; b < kb; ++b)
      if ((uint32_t)J.lo_mask >> b & 1u) lo_of |= (uint32_t)(kb + nlo++ + 1) << (8 * b);
    const int64_t mt = (J.h1 + kBM - 1) / kBM, nt = (J.h2 + kBN - 1) / kBN;
    // loads move whole 128-row boxes; each epilogue warp stores its own 32 rows
    if (int rc = make_w_map(&maps[4 * j], J.w_in, J.h1, J.h2, J.ldw, kBM)) return rc;
    if (int rc = make_w_map(&maps[4 * j + 1], J.w_out, J.h1, J.h2, J.ldw, 32)) return rc;
    if (int rc = make_f_map(&maps[4 * j + 2], J.a_packed, mt * kb * kBM)) return rc;
    if (int rc = make_f_map(&maps[4 * j + 3], J.b_packed, nt * (kb + nlo) * kBN)) return rc;
    std::memset(&tj[j], 0, sizeof(TcJob));
    tj[j].a = static_cast<const uint8_t*>(J.a_packed);
    tj[j].b = static_cast<const uint8_t*>(J.b_packed);
    tj[j].h1 = J.h1;
    tj[j].h2 = J.h2;
    tj[j].kb = kb;
    tj[j].rank = J.rank;
    tj[j].scale = J.scale;
    tj[j].map_in = 4 * j;
    tj[j].map_out = 4 * j + 1;
    tj[j].map_a = 4 * j + 2;
    tj[j].map_b = 4 * j + 3;
    tj[j].mt = (int32_t)mt;
    tj[j].bkb = kb + nlo;
    tj[j].lo_of = lo_of;
  }
  std::memcpy(base + maps_b + jobs_b, units.data(), units_b);
  return SDB_OK;
}

int tc_set_mode(int mode) {
  if (mode < 0 || mode > 2) return fail(SDB_EINVAL, "lora_tc_set_mode: mode must be 0 (auto), 1 (single CTA) or 2 (CTA pair)");
  const int prev = g_tc_mode;
  g_tc_mode = mode;
  return prev;
}

int tc_patch(const void* blob_dev, int n_jobs, int n_units, int kb_word, int simt_rank, float sign, int max_ctas,
             cudaStream_t st) {
  // kb_max: B-panel K-blocks (sizes the resident panel); akb_max: A K-blocks (the A ring)
  const int kb_max = kb_word & 0xFF, mode = (kb_word >> 8) & 0xF, akb_max = std::max(1, kb_word >> 12);
  if (!blob_dev || n_units <= 0) return fail(SDB_EINVAL, "lora_tc_patch: empty plan");
  if (((uintptr_t)blob_dev) & 127) return fail(SDB_EINVAL, "lora_tc_patch: blob must be 128-B aligned");
  if (kb_max < 1 || kb_max > 2 * kMaxKB) return fail(SDB_EINVAL, "lora_tc_patch: kb_max out of range");
  if (mode != 1 && mode != 2) return fail(SDB_EINVAL, "lora_tc_patch: kb_max word is not from sdb_lora_tc_plan");
  const size_t maps_b = (size_t)4 * n_jobs * sizeof(CUtensorMap);
  const uint8_t* base = static_cast<const uint8_t*>(blob_dev);
  const CUtensorMap* maps = reinterpret_cast<const CUtensorMap*>(base);
  const TcJob* jobs = reinterpret_cast<const TcJob*>(base + maps_b);
  const TcUnit* units = reinterpret_cast<const TcUnit*>(base + maps_b + (size_t)n_jobs * sizeof(TcJob));
  (void)simt_rank;  // reserved (ABI): the FFMA variant was retired, tcgen05 wins at every rank (profiles/)
  const int max_smem = 227 * 1024;
  if (mode == 2) {
    // A K-blocks in flight = the K blocks of one tile (2..4): a tile's MMAs
    // consume them in sequence, so at high rank a deeper A ring beats the
    // last W slots (round 1, R = 232: 4 stages + 6 slots 2.04 ms = 89% of the
    // copy peak vs 2 stages + 8 slots 2.42 ms; R <= 128: 2 stages best)
    // with low-part B blocks the panel grows (R = 232, four scales: 6 blocks);
    // 3 A stages leave 5 W slots — measured best (2 / 3 / 4 stages: 2.64 /
    // 2.46 / 2.78 ms, all 794 SDXL matrices, scripts/k1_scales_probe.py)
    const int na = kb_max > akb_max ? 3 : std::min(4, std::max(2, akb_max));
    const int fixed = 1024 + kb_max * kHalfBlock + na * kABlockBytes + 320;
    const int slots = std::min(kMaxSlots, (max_smem - fixed) / kBoxBytes);
    const int smem = fixed + slots * kBoxBytes;
    cudaFuncSetAttribute(lora_patch_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    // persistent grid = the CTA pairs that can be co-resident (TPCs usable by
    // 2-CTA clusters); launching more would leave a second wave doing the tail
    static int s_pairs = 0, s_smem = -1;
    if (s_smem != smem) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(kNumSMs & ~1, 1, 1);
      cfg.blockDim = dim3(kThreads, 1, 1);
      cfg.dynamicSmemBytes = smem;
      int n = 0;
      if (cudaOccupancyMaxActiveClusters(&n, lora_patch_pair_kernel, &cfg) != cudaSuccess || n <= 0) {
        cudaGetLastError();
        n = kNumSMs / 2;
      }
      s_pairs = std::min(n, kNumSMs / 2);
      s_smem = smem;
      if (getenv("SDB_DEBUG")) fprintf(stderr, "sdb: lora_patch_pair_kernel smem %d B, co-resident pairs %d\n", smem, n);
    }
    int grid = std::min(2 * n_units, 2 * s_pairs);
    if (max_ctas > 0) grid = std::min(grid, std::max(2, max_ctas));
    grid &= ~1;
    lora_patch_pair_kernel<<<grid, kThreads, smem, st>>>(maps, jobs, units, n_units, sign, kb_max, slots, na);
    return check_launch("lora_patch_pair_kernel");
  }
  const int fixed = 1024 + kb_max * kBN * 128 + kAStages * kABlockBytes + 256;
  int slots = std::min(8, (max_smem - fixed) / kBoxBytes);
  if (slots < 2) return fail(SDB_EUNSUP, "lora_tc_patch: rank too large for shared memory");
  const int smem = fixed + slots * kBoxBytes;
  int grid = std::min(n_units, kNumSMs);
  if (max_ctas > 0) grid = std::min(grid, max_ctas);
  cudaFuncSetAttribute(lora_patch_tma_kernel<kBN>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  lora_patch_tma_kernel<kBN><<<grid, kThreads, smem, st>>>(maps, jobs, units, n_units, sign, kb_max, slots);
  return check_launch("lora_patch_tma_kernel");
}

}  // namespace sdb
