// self_attn.cu — K8: the UNet's self-attention (head dim 64, non-causal) on
// tcgen05, flash-style: one CTA = 128 queries of one (sample, head) walking
// the sequence in 128-key blocks with an online softmax.
//
//   qkv: [N, L, 3C] rows of stride ldqkv (the fused to_q|to_k|to_v GEMM output:
//        Q at column h*64, K at C + h*64, V at 2C + h*64), o: [N, L, C] rows of
//        stride ldo, C = H * 64, L % 128 == 0.
//
// Roles: warps 0-3 own one query row per thread (= TMEM lane); warp 4 lane 0
// issues the TMA loads and the MMAs.  Per key block j:
//   S_j = Q K_j^T            tcgen05.mma M128 x N128 x K64 -> TMEM cols [0,128)
//   row max (two 64-column TMEM passes), p = 2^(s*c - m), P_j (bf16) -> a
//   128-B-swizzled smem A tile, running sum l, rescale alpha_j = 2^(m_{j-1}-m_j)
//   PV_j = P_j V_j           M128 x N64 x K128 (V as stored: MN-major B)
//                            -> TMEM cols [128 + 64 (j & 1), ...)
//   O (registers) = O * alpha_{j} + PV_j once PV_j is done (during block j+1)
// K/V blocks are double-buffered by TMA; PV_j runs under softmax j+1.
// Status: correct (tests/test_kernels_gpu.py) but not faster than the library
// cuDNN kernel at SDXL's shapes, so the UNet keeps SDPA unless SDB_SELF_ATTN=1.
// Round 1 (single-S kernel below, SDB_FMHA=1): L=1024 32 vs 25 us, L=4096 169
// vs 122 us.  Round 2 (fmha2_kernel, default): 28.5 / 144 us
// (scripts/fmha2_probe.py, profiles/r02_k8_probes.txt).  What bounds it: the
// softmax phase is MUFU-bound (16 ex2/clk/SM; per-block trace ~96% busy),
// ~330 clocks of barrier hand-offs per 64-key block, and the grid: 640 tiles
// over 296 resident CTAs = 3 rounds where 2.16 are needed (320 over 296 = 2
// rounds for 1.08 at L = 1024).  Measured dead ends: ex2 on the FMA pipe
// (degree-3 polynomial for 1/4 or 1/2 of the scores: slower), 32-key blocks
// with 3 CTAs/SM (one round at L = 1024: 28.2 us), a stream-K split of the
// (tile, key block) units with last-arriver combines (46 / 194 us: the
// combine chains cost more than the tail they remove), two query tiles per
// CTA sharing K/V (217-230 us).  The reference has no attention arithmetic
// (addonsim is a latency model): this kernel is part of the UNet backbone
// the denoising loop runs, replacing the library SDPA call of a
// diffusers-style Attention.
#include <cuda.h>

#include <cstdlib>

#include "common.cuh"
#include "ptx.cuh"
#include "tcgen05.cuh"

namespace sdb {
namespace {

constexpr int kM = 128;        // queries per CTA (TMEM lanes)
constexpr int kBK = 128;       // keys per block
constexpr int kThreads = 160;  // 4 softmax warps + 1 control warp
constexpr int kTile = 128 * 128;   // one 128-row x 128-B swizzled tile (16 KB)

__device__ __forceinline__ float ex2f(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// 2^t for a pair on the FMA pipe (the MUFU does 16 ex2/clk/SM; a share of the
// softmax's exponentials moves here): t = n + f, n = round(t) via the 1.5*2^23
// trick, 2^f on [-0.5, 0.5] by a degree-3 minimax polynomial (max relative
// error 7.5e-5, far below bf16's 2^-9), n added to the exponent field (the
// magic's own bits vanish in the shift).  t is clamped at -125 (2^-125 ~ 0).
__device__ __forceinline__ float2 ex2_fma2(float2 t) {
  t = make_float2(fmaxf(t.x, -125.f), fmaxf(t.y, -125.f));
  const float2 r = f2add(t, f2s(12582912.f));
  const float2 k = f2add(r, f2s(-12582912.f));
  const float2 f = f2fma(k, f2s(-1.f), t);
  float2 q = f2fma(f2s(0.055171653628349304f), f, f2s(0.24261115491390228f));
  q = f2fma(q, f, f2s(0.6932609677314758f));
  q = f2fma(q, f, f2s(0.9999280571937561f));
  return make_float2(__int_as_float(__float_as_int(q.x) + (__float_as_int(r.x) << 23)),
                     __int_as_float(__float_as_int(q.y) + (__float_as_int(r.y) << 23)));
}
__device__ __forceinline__ uint32_t pk_bf16(float lo, float hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}
__global__ void __launch_bounds__(kThreads, 2)
fmha_tc_kernel(const __grid_constant__ CUtensorMap map, __nv_bfloat16* __restrict__ o, int64_t ldo, int L, int C,
               float scale_log2) {
  constexpr uint32_t kIdescS = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kBK >> 3) << 17) |
                               ((uint32_t)(kM >> 4) << 24);
  constexpr uint32_t kIdescO = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) | ((uint32_t)(64 >> 3) << 17) |
                               ((uint32_t)(kM >> 4) << 24);
  // [barriers | pad to 1024] [Q 16 KB] [2 x (K 16 KB | V 16 KB)] [P 2 x 16 KB]: 115,712 B, so two
  // CTAs (+1 KB reserved each) fit the SM's 228 KB
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw);
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 128 + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;                         // 16 KB
  uint8_t* sKV = smem + kTile;                // 2 stages x (K 16 KB | V 16 KB)
  uint8_t* sP = sKV + 4 * kTile;              // P: 2 atoms (keys 0-63 | 64-127) x 16 KB
  // barriers
  const int KV_FULL = 0, KV_EMPTY = 2, S_FULL = 4, S_EMPTY = 5, P_FULL = 6, PV_FULL = 7, PV_EMPTY = 9;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 11);
  auto bar = [&](int i) { return smem_u32(bars + i); };

  const int h = blockIdx.y, n = blockIdx.z, q0 = blockIdx.x * kM;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int nblk = L / kBK;
  const int row0 = n * L;                     // first row of this sample in the qkv map

  if (tid == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(bar(KV_FULL + i), 1);
      mbar_init(bar(KV_EMPTY + i), 1);
      mbar_init(bar(PV_FULL + i), 1);
      mbar_init(bar(PV_EMPTY + i), kM);
    }
    mbar_init(bar(S_FULL), 1);
    mbar_init(bar(S_EMPTY), kM);
    mbar_init(bar(P_FULL), kM);
    mbar_fence_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                 "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;

  if (warp == 4) {
    // ======================= control: TMA + MMA issue =======================
    if ((tid & 31) == 0) {
      const uint64_t keep = policy_evict_last();
      auto load_kv = [&](int j, int st) {
        uint8_t* k = sKV + st * 2 * kTile;
        tma_load_2d(smem_u32(k), &map, C + h * 64, row0 + j * kBK, bar(KV_FULL + st), keep);
        tma_load_2d(smem_u32(k + kTile), &map, 2 * C + h * 64, row0 + j * kBK, bar(KV_FULL + st), keep);
      };
      mbar_expect_tx(bar(KV_FULL), 3 * kTile);
      tma_load_2d(smem_u32(sQ), &map, h * 64, row0 + q0, bar(KV_FULL), policy_evict_first());
      load_kv(0, 0);
      if (nblk > 1) {
        mbar_expect_tx(bar(KV_FULL + 1), 2 * kTile);
        load_kv(1, 1);
      }
      auto issue_pv = [&](int j) {   // PV_j = P_j V_j into PV buffer j & 1
        mbar_wait(bar(P_FULL), j & 1);
        if (j >= 2) mbar_wait(bar(PV_EMPTY + (j & 1)), ((j >> 1) - 1) & 1);
        tc_fence_after();
        const uint32_t d = tmem + 128 + 64 * (j & 1);
        const uint8_t* v = sKV + (j & 1) * 2 * kTile + kTile;
#pragma unroll
        for (int ks = 0; ks < kBK / 16; ++ks)
          tc_mma(d, sw128_desc(smem_u32(sP) + (ks >> 2) * kTile + (ks & 3) * 32), sw128_desc(smem_u32(v) + ks * 2048),
                 kIdescO, ks ? 1u : 0u);
        tc_commit(bar(PV_FULL + (j & 1)));
        tc_commit(bar(KV_EMPTY + (j & 1)));
      };
      for (int j = 0; j < nblk; ++j) {
        const int st = j & 1;
        mbar_wait(bar(KV_FULL + st), (j >> 1) & 1);
        if (j >= 1) mbar_wait(bar(S_EMPTY), (j - 1) & 1);
        tc_fence_after();
        const uint8_t* k = sKV + st * 2 * kTile;
#pragma unroll
        for (int ks = 0; ks < 4; ++ks)
          tc_mma(tmem, sw128_desc(smem_u32(sQ) + ks * 32), sw128_desc(smem_u32(k) + ks * 32), kIdescS, ks ? 1u : 0u);
        tc_commit(bar(S_FULL));
        if (j >= 1) {
          issue_pv(j - 1);
          // stage (j-1)&1 is free once PV_{j-1} has read V_{j-1}: refill it with block j+1
          if (j + 1 < nblk) {
            mbar_wait(bar(KV_EMPTY + ((j - 1) & 1)), ((j - 1) >> 1) & 1);
            mbar_expect_tx(bar(KV_FULL + ((j + 1) & 1)), 2 * kTile);
            load_kv(j + 1, (j + 1) & 1);
          }
        }
      }
      issue_pv(nblk - 1);
    }
    __syncwarp();
  } else {
    // ======================= softmax: one query row per thread ==============
    const uint32_t lane_s = tmem + ((uint32_t)(warp * 32) << 16);
    float O[64];
#pragma unroll
    for (int i = 0; i < 64; ++i) O[i] = 0.f;
    float m_old = -INFINITY, l = 0.f, alpha_prev = 1.f;
    uint8_t* prow = sP + tid * 128;
    const int sw = tid & 7;
    for (int j = 0; j < nblk; ++j) {
      mbar_wait(bar(S_FULL), j & 1);
      tc_fence_after();
      // pass 1: row max over the block's 128 scores
      float mx = m_old;
#pragma unroll
      for (int q4 = 0; q4 < 4; ++q4) {
        float v[32];
        tc_ld32(lane_s + 32 * q4, v);
#pragma unroll
        for (int i = 0; i < 32; ++i) mx = fmaxf(mx, v[i]);
      }
      const float mb = mx * scale_log2;
      const float alpha = ex2f((m_old - mx) * scale_log2);   // 0 on the first block (m_old = -inf)
      // P_j overwrites P_{j-1}: PV_{j-1} must have read it
      if (j >= 1) mbar_wait(bar(PV_FULL + ((j - 1) & 1)), ((j - 1) >> 1) & 1);
      // pass 2: p = 2^(s c - m c), row sum, bf16 into the swizzled A tile
      float rs = 0.f;
#pragma unroll
      for (int q4 = 0; q4 < 4; ++q4) {        // 32 keys = 4 16-B chunks of the row at a time
        float v[32];
        tc_ld32(lane_s + 32 * q4, v);
#pragma unroll
        for (int c4 = 0; c4 < 4; ++c4) {
          float p[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            p[e] = ex2f(fmaf(v[8 * c4 + e], scale_log2, -mb));
            rs += p[e];
          }
          uint4 pk;
          pk.x = pk_bf16(p[0], p[1]);
          pk.y = pk_bf16(p[2], p[3]);
          pk.z = pk_bf16(p[4], p[5]);
          pk.w = pk_bf16(p[6], p[7]);
          const int c8 = (q4 & 1) * 4 + c4;   // 16-B chunk within the 64-key atom
          *reinterpret_cast<uint4*>(prow + (q4 >> 1) * kTile + ((c8 ^ sw) << 4)) = pk;
        }
      }
      tc_fence_before();
      mbar_arrive(bar(S_EMPTY));          // S_j fully read: the next S may overwrite it
      fence_proxy_async();
      mbar_arrive(bar(P_FULL));
      // fold PV_{j-1} (complete: waited above) into O
      if (j >= 1) {
        tc_fence_after();
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          float pv[32];
          tc_ld32(tmem + 128 + 64 * ((j - 1) & 1) + 32 * hh + ((uint32_t)(warp * 32) << 16), pv);
#pragma unroll
          for (int i = 0; i < 32; ++i) O[32 * hh + i] = fmaf(O[32 * hh + i], alpha_prev, pv[i]);
        }
        tc_fence_before();
        mbar_arrive(bar(PV_EMPTY + ((j - 1) & 1)));
      }
      l = fmaf(l, alpha, rs);
      alpha_prev = alpha;
      m_old = mx;
    }
    // the last block's PV
    mbar_wait(bar(PV_FULL + ((nblk - 1) & 1)), ((nblk - 1) >> 1) & 1);
    tc_fence_after();
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      float pv[32];
      tc_ld32(tmem + 128 + 64 * ((nblk - 1) & 1) + 32 * hh + ((uint32_t)(warp * 32) << 16), pv);
#pragma unroll
      for (int i = 0; i < 32; ++i) O[32 * hh + i] = fmaf(O[32 * hh + i], alpha_prev, pv[i]);
    }
    float rl;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rl) : "f"(l));
    __nv_bfloat16* orow = o + ((int64_t)n * L + q0 + tid) * ldo + h * 64;
#pragma unroll
    for (int c8 = 0; c8 < 8; ++c8) {
      uint4 pk;
      pk.x = pk_bf16(O[8 * c8 + 0] * rl, O[8 * c8 + 1] * rl);
      pk.y = pk_bf16(O[8 * c8 + 2] * rl, O[8 * c8 + 3] * rl);
      pk.z = pk_bf16(O[8 * c8 + 4] * rl, O[8 * c8 + 5] * rl);
      pk.w = pk_bf16(O[8 * c8 + 6] * rl, O[8 * c8 + 7] * rl);
      *reinterpret_cast<uint4*>(orow + c8 * 8) = pk;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
  }
}


// ---- K8 v2: S double-buffered in TMEM, O accumulated in TMEM ----------------
// One CTA = 128 queries of one (sample, head); 64-key blocks; warps 0-3
// softmax (thread = query row = TMEM lane), warp 4 TMA producer, warp 5 MMA
// issuer; two CTAs per SM.  TMEM (256 columns): S0 [0,64), S1 [64,128), O
// [128,192).  The MMA warp issues S(j+1) BEFORE PV(j), so the tensor core
// computes the next block's scores while the softmax warps work on this
// block's: the softmax never waits on the tensor core in steady state (round
// 1's kernel did, every block: one S buffer).  P(j) goes to one of two
// swizzled smem tiles; O += P(j) V(j) accumulates in TMEM (no per-block fold
// through registers).  Softmax: one TMEM pass per block against a reference
// max m_ref (log2 units, the first block's max) and no per-score max at all:
// every p is at most the row's block sum, so a sum <= 2^16 proves every p is
// exact in fp32 and representable in bf16; a larger (or non-finite) sum
// raises the reference to that row's block max (warp-uniformly: the block is
// recomputed, O (TMEM) and l rescaled by 2^(old - new)).  Packed f32x2 FFMA /
// FADD: ~2.6 issued instructions per score.  Per-block trace
// (scripts/fmha_trace.py probe build, L = 4096): ~1070 clocks of softmax —
// the MUFU (16 ex2/clk/SM, shared by the SM's two CTAs) busy ~96% of it —
// plus ~330 clocks of hand-offs per 64-key block.
constexpr int kF2Threads = 192;
constexpr int kF2Stages = 3;                   // K|V stages
constexpr float kF2SumCap = 65536.f;           // lazy rescale: a block row sum above 2^16 raises the reference

__device__ __forceinline__ void tc_ld32_raw(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tc_st32_raw(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
      "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
      "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
__device__ __forceinline__ void tc_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tc_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

template <int BK, int EMU>   // keys per block: 64 (2 CTAs/SM) or 32 (3 CTAs/SM); EMU: ex2 pairs per 4 on the FMA pipe
__global__ void __launch_bounds__(kF2Threads, BK == 32 ? 3 : 2)
fmha2_kernel(const __grid_constant__ CUtensorMap qmap, const __grid_constant__ CUtensorMap kvmap,
             __nv_bfloat16* __restrict__ o, int64_t ldo, int L, int C, float scale_log2) {
  constexpr int kF2BK = BK;
  constexpr int kF2KV = BK * 128;               // one K (or V) block: BK rows x 128 B
  constexpr uint32_t kTmemCols = BK == 32 ? 128 : 256;   // S0 | S1 | O (64)
  constexpr uint32_t kIdescS = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kF2BK >> 3) << 17) |
                               ((uint32_t)(kM >> 4) << 24);
  constexpr uint32_t kIdescO = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) | ((uint32_t)(64 >> 3) << 17) |
                               ((uint32_t)(kM >> 4) << 24);
  // [barriers | pad] [Q 16 KB] [kF2Stages x (K | V) 16 KB] [P0 | P1 2 x 16 KB]
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw);
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 256 + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sKV = smem + kTile;                      // stage s: K at + s * 2 * kF2KV, V at + kF2KV
  uint8_t* sP = sKV + kF2Stages * 2 * kF2KV;        // buffer b at + b * kTile
  const int Q_FULL = 0, KV_FULL = 1, KV_EMPTY = KV_FULL + kF2Stages, S_FULL = KV_EMPTY + kF2Stages,
            S_EMPTY = S_FULL + 2, P_FULL = S_EMPTY + 2, PV_DONE = P_FULL + 2;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + PV_DONE + 2);
  auto bar = [&](int i) { return smem_u32(bars + i); };

  const int h = blockIdx.y, n = blockIdx.z, q0 = blockIdx.x * kM;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int nblk = L / kF2BK;
  const int row0 = n * L;

  if (tid == 0) {
    mbar_init(bar(Q_FULL), 1);
    for (int i = 0; i < kF2Stages; ++i) {
      mbar_init(bar(KV_FULL + i), 1);
      mbar_init(bar(KV_EMPTY + i), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(bar(S_FULL + b), 1);
      mbar_init(bar(S_EMPTY + b), kM);
      mbar_init(bar(P_FULL + b), kM);
      mbar_init(bar(PV_DONE + b), 1);
    }
    mbar_fence_init();
    prefetch_map(&qmap);
    prefetch_map(&kvmap);
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  pdl_wait();

  if (warp == 4) {
    // ============================ TMA producer ===============================
    if ((tid & 31) == 0) {
      const uint64_t keep = policy_evict_last();
      mbar_expect_tx(bar(Q_FULL), kTile);
      tma_load_2d(smem_u32(sQ), &qmap, h * 64, row0 + q0, bar(Q_FULL), policy_evict_first());
      for (int j = 0; j < nblk; ++j) {
        const int st = j % kF2Stages;
        if (j >= kF2Stages) mbar_wait(bar(KV_EMPTY + st), ((j / kF2Stages) - 1) & 1);
        uint8_t* k = sKV + st * 2 * kF2KV;
        mbar_expect_tx(bar(KV_FULL + st), 2 * kF2KV);
        tma_load_2d(smem_u32(k), &kvmap, C + h * 64, row0 + j * kF2BK, bar(KV_FULL + st), keep);
        tma_load_2d(smem_u32(k + kF2KV), &kvmap, 2 * C + h * 64, row0 + j * kF2BK, bar(KV_FULL + st), keep);
      }
    }
    __syncwarp();
  } else if (warp == 5) {
    // ============================ MMA issuer =================================
    if ((tid & 31) == 0) {
      auto issue_s = [&](int j) {
        const int b = j & 1;
        const uint8_t* k = sKV + (j % kF2Stages) * 2 * kF2KV;
#pragma unroll
        for (int ks = 0; ks < 4; ++ks)
          tc_mma(tmem + BK * b, sw128_desc(smem_u32(sQ) + ks * 32), sw128_desc(smem_u32(k) + ks * 32), kIdescS,
                 ks ? 1u : 0u);
        tc_commit(bar(S_FULL + b));
      };
      mbar_wait(bar(Q_FULL), 0);
      mbar_wait(bar(KV_FULL), 0);
      tc_fence_after();
      issue_s(0);
      for (int j = 0; j < nblk; ++j) {
        if (j + 1 < nblk) {   // S(j+1) first: computed while the softmax works on S(j)
          mbar_wait(bar(KV_FULL + (j + 1) % kF2Stages), ((j + 1) / kF2Stages) & 1);
          if (j + 1 >= 2) mbar_wait(bar(S_EMPTY + ((j + 1) & 1)), (((j + 1) >> 1) - 1) & 1);
          tc_fence_after();
          issue_s(j + 1);
        }
        const int b = j & 1;
        mbar_wait(bar(P_FULL + b), (j >> 1) & 1);
        tc_fence_after();
        const uint8_t* v = sKV + (j % kF2Stages) * 2 * kF2KV + kF2KV;
#pragma unroll
        for (int ks = 0; ks < kF2BK / 16; ++ks)
          tc_mma(tmem + 2 * BK, sw128_desc(smem_u32(sP + b * kTile) + ks * 32), sw128_desc(smem_u32(v) + ks * 2048),
                 kIdescO, (j > 0 || ks > 0) ? 1u : 0u);
        tc_commit(bar(PV_DONE + b));
        tc_commit(bar(KV_EMPTY + j % kF2Stages));
      }
    }
    __syncwarp();
  } else {
    // ===================== softmax: one query row per thread =================
    const int r = tid;                          // row = TMEM lane
    const uint32_t lane = (uint32_t)(warp * 32) << 16;
    const uint32_t o_addr = tmem + 2 * BK + lane;
    float m_ref = 0.f, l = 0.f;
    const int sw = r & 7;
    for (int j = 0; j < nblk; ++j) {
      const int b = j & 1;
      const uint32_t s_addr = tmem + BK * b + lane;
      mbar_wait(bar(S_FULL + b), (j >> 1) & 1);
      tc_fence_after();
      if (j == 0) {   // the first block fixes the reference max
        float mx = -INFINITY;
#pragma unroll
        for (int q4 = 0; q4 < BK / 32; ++q4) {
          uint32_t v[32];
          tc_ld32_raw(s_addr + 32 * q4, v);
          tc_wait_ld();
#pragma unroll
          for (int i = 0; i < 32; ++i) mx = fmaxf(mx, __uint_as_float(v[i]));
        }
        m_ref = mx * scale_log2;
      }
      if (j >= 2) mbar_wait(bar(PV_DONE + b), ((j >> 1) - 1) & 1);   // P buffer b free (PV(j-2) done)
      uint8_t* prow = sP + b * kTile + r * 128;
      // p = 2^(s c - m_ref) for the block's scores -> P (bf16, swizzled smem), returns the row sum.
      // Packed f32x2 FFMA / FADD: ~2.6 issued instructions per score (round 1: ~5.5).
      const float2 sc2 = f2s(scale_log2);
      auto exp_pass = [&]() -> float {
        const float2 nm2 = f2s(-m_ref);
        float2 rs2 = f2s(0.f);
#pragma unroll
        for (int q4 = 0; q4 < BK / 32; ++q4) {
          uint32_t v[32];
          tc_ld32_raw(s_addr + 32 * q4, v);
          tc_wait_ld();
#pragma unroll
          for (int c4 = 0; c4 < 4; ++c4) {
            uint32_t pk[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float2 x = make_float2(__uint_as_float(v[8 * c4 + 2 * e]), __uint_as_float(v[8 * c4 + 2 * e + 1]));
              const float2 t = f2fma(x, sc2, nm2);
              const float2 pe = e < EMU ? ex2_fma2(t) : make_float2(ex2f(t.x), ex2f(t.y));
              rs2 = f2add(rs2, pe);
              pk[e] = pk_bf16(pe.x, pe.y);
            }
            const int c8 = q4 * 4 + c4;
            *reinterpret_cast<uint4*>(prow + ((c8 ^ sw) << 4)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
          }
        }
        return rs2.x + rs2.y;
      };
      float alpha = 1.f;
      float rs = exp_pass();
      // no per-score max in the common pass: every p <= the row sum, so a sum <= 2^16 bounds every p
      // (exact in fp32, representable in bf16); a larger (or non-finite) sum -> this row's block max,
      // raise the reference, recompute (warp-uniform: tcgen05.ld is .sync.aligned)
      const bool need = !(rs <= kF2SumCap);
      if (__any_sync(0xffffffffu, need)) {
        float mx = -INFINITY;
#pragma unroll
        for (int q4 = 0; q4 < BK / 32; ++q4) {
          uint32_t v[32];
          tc_ld32_raw(s_addr + 32 * q4, v);
          tc_wait_ld();
#pragma unroll
          for (int i = 0; i < 32; ++i) mx = fmaxf(mx, __uint_as_float(v[i]));
        }
        if (need) {
          const float bm = mx * scale_log2;
          alpha = ex2f(m_ref - bm);
          m_ref = bm;
        }
        rs = exp_pass();
      }
      tc_fence_before();
      mbar_arrive(bar(S_EMPTY + b));
      if (__any_sync(0xffffffffu, alpha != 1.f)) {   // rescale O = sum of PV(0..j-1): PV(j-1) must be done
        mbar_wait(bar(PV_DONE + (b ^ 1)), ((j - 1) >> 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          uint32_t v[32];
          tc_ld32_raw(o_addr + 32 * hh, v);
          tc_wait_ld();
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * alpha);
          tc_st32_raw(o_addr + 32 * hh, v);
        }
        tc_wait_st();
        tc_fence_before();
      }
      fence_proxy_async();
      mbar_arrive(bar(P_FULL + b));
      l = fmaf(l, alpha, rs);
    }
    mbar_wait(bar(PV_DONE + ((nblk - 1) & 1)), ((nblk - 1) >> 1) & 1);
    tc_fence_after();
    float rl;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rl) : "f"(l));
    __nv_bfloat16* orow = o + ((int64_t)n * L + q0 + r) * ldo + h * 64;
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      uint32_t v[32];
      tc_ld32_raw(o_addr + 32 * hh, v);
      tc_wait_ld();
#pragma unroll
      for (int c8 = 0; c8 < 4; ++c8) {
        uint4 pk;
        pk.x = pk_bf16(__uint_as_float(v[8 * c8 + 0]) * rl, __uint_as_float(v[8 * c8 + 1]) * rl);
        pk.y = pk_bf16(__uint_as_float(v[8 * c8 + 2]) * rl, __uint_as_float(v[8 * c8 + 3]) * rl);
        pk.z = pk_bf16(__uint_as_float(v[8 * c8 + 4]) * rl, __uint_as_float(v[8 * c8 + 5]) * rl);
        pk.w = pk_bf16(__uint_as_float(v[8 * c8 + 6]) * rl, __uint_as_float(v[8 * c8 + 7]) * rl);
        *reinterpret_cast<uint4*>(orow + 32 * hh + c8 * 8) = pk;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
  }
}

}  // namespace

int self_attention(const void* qkv, int64_t ldqkv, void* o, int64_t ldo, int n, int L, int heads, int head_dim,
                   float scale, int dtype, cudaStream_t st) {
  if (dtype != SDB_BF16) return fail(SDB_EUNSUP, "self_attention: bf16 only");
  if (head_dim != 64) return fail(SDB_EUNSUP, "self_attention: head dim 64 only");
  if (n <= 0 || heads <= 0 || L <= 0 || L % kBK != 0) return fail(SDB_EUNSUP, "self_attention: L must be a multiple of 128");
  const int C = heads * 64;
  if (ldqkv < 3 * C || ldo < C || (ldqkv | ldo) % 8) return fail(SDB_EINVAL, "self_attention: bad row strides");
  if (((uintptr_t)qkv | (uintptr_t)o) & 15) return fail(SDB_EINVAL, "self_attention: pointers must be 16-B aligned");
  EncodeTiledFn enc = encode_fn();
  if (!enc) return fail(SDB_ECUDA, "cuTensorMapEncodeTiled unavailable");
  CUtensorMap map;
  cuuint64_t dims[2] = {(cuuint64_t)(3 * C), (cuuint64_t)n * L};
  cuuint64_t strides[1] = {(cuuint64_t)ldqkv * 2};
  cuuint32_t box[2] = {64, 128};
  cuuint32_t es[2] = {1, 1};
  if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(qkv), dims, strides, box, es,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return fail(SDB_EINVAL, "self_attention: tensor map");
  static int mode = -1;   // SDB_FMHA=1: round 1's single-tile kernel
  if (mode < 0) mode = getenv("SDB_FMHA") != nullptr ? atoi(getenv("SDB_FMHA")) : 2;
  if (mode == 2) {
    // 64-key blocks, 2 CTAs/SM; SDB_FMHA_BK=32: 32-key blocks, 3 CTAs/SM (444 resident tiles: one
    // round at L = 1024) — measured 28.2 vs 28.5 us there, 162.5 vs 144.4 us at L = 4096
    static int bk = -1;
    if (bk < 0) bk = getenv("SDB_FMHA_BK") != nullptr ? atoi(getenv("SDB_FMHA_BK")) : 64;
    const int smem2 = 256 + 1024 + kTile + kF2Stages * 2 * bk * 128 + 2 * kTile;   // 72,960 / 99,584 B
    // SDB_FMHA_EMU: exponential pairs per 4 on the FMA pipe (ex2_fma2); 0 (default): measured
    // 144.4 / 28.5 us at [2,4096,10] / [2,1024,20] vs 151.6 / 29.5 (1) and 152.8 / 30.1 (2)
    static int emu = -1;
    if (emu < 0) emu = getenv("SDB_FMHA_EMU") != nullptr ? atoi(getenv("SDB_FMHA_EMU")) : 0;
    auto kern = bk == 64 ? (emu == 0 ? fmha2_kernel<64, 0> : emu == 2 ? fmha2_kernel<64, 2> : fmha2_kernel<64, 1>)
                         : (emu == 0 ? fmha2_kernel<32, 0> : emu == 2 ? fmha2_kernel<32, 2> : fmha2_kernel<32, 1>);
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem2);
    CUtensorMap kvm;
    cuuint32_t box2[2] = {64, (cuuint32_t)bk};
    if (enc(&kvm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(qkv), dims, strides, box2, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return fail(SDB_EINVAL, "self_attention: tensor map");
    dim3 grid2((unsigned)(L / kM), (unsigned)heads, (unsigned)n);
    launch_k(kern, grid2, kF2Threads, smem2, st, map, kvm, static_cast<__nv_bfloat16*>(o), ldo, L, C,
             scale * 1.4426950408889634f);
    return check_launch("fmha2_kernel");
  }
  const int smem = 1024 + 7 * kTile;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(fmha_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  dim3 grid((unsigned)(L / kM), (unsigned)heads, (unsigned)n);
  fmha_tc_kernel<<<grid, kThreads, smem, st>>>(map, static_cast<__nv_bfloat16*>(o), ldo, L, C,
                                               scale * 1.4426950408889634f);
  return check_launch("fmha_tc_kernel");
}

}  // namespace sdb
