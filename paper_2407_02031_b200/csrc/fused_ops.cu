// fused_ops.cu — memory-bound fusions around the transformer blocks of the
// UNet / ControlNet (HBM-bound: one read of each input, one write of each output).
//
// K5 geglu:          out[m, :] = h[m, :] * gelu(g[m, :]),  [h | g] = proj[m, 0:2F]
//                    (the paper's fused GEGLU, PAPER.md:567-570, 70 sites in
//                    SDXL; the reference keeps only its 1.06 sub-multiplier,
//                    addonsim/model.py:66-70).  Exact erf GELU as torch's default.
// K6 add_layernorm:  x[m, :] += d[m, :] (d optional; written back in place), then
//                    y[m, :] = LayerNorm(x[m, :]) * gamma + beta (eps 1e-5),
//                    replacing torch's residual add + LayerNorm pair (two extra
//                    round trips of the residual stream per block).
// One warp per row (C up to 2560 for LN); fp32 statistics, two-pass over the
// row held in registers.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "ptx.cuh"
#include "tcgen05.cuh"

namespace sdb {
namespace {

// Each thread owns kGegluVec 8-element vectors spaced one grid apart and issues
// all of their loads (value and gate halves) before computing any.
constexpr int kGegluVec = 4;

// GELU(g) = g * Phi(g) on a pair of values with packed fp32x2 arithmetic.
// Phi comes from erf by Abramowitz & Stegun 7.1.26 (|error| <= 1.5e-7 in erf,
// i.e. at fp32 rounding level and far below the bf16 output ulp), rearranged so
// that no branch is needed and the negative tail has no cancellation:
//   GELU(g) = 0.5 (g + |g|) - 0.5 |g| P(t) exp(-g^2 / 2),  t = 1 / (1 + p |g| / sqrt 2)
// Two MUFU ops (rcp, ex2) and ~11 packed instructions per pair instead of the
// libdevice erff's ~25 scalar instructions and two divergent paths per value.
__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float ex2_approx(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float2 gelu2(float2 g) {
  constexpr float kP = 0.3275911f * 0.70710678118654752f;     // p / sqrt(2)
  // A&S coefficients a1..a5 scaled by -0.5
  constexpr float b1 = -0.5f * 0.254829592f, b2 = -0.5f * -0.284496736f, b3 = -0.5f * 1.421413741f,
                  b4 = -0.5f * -1.453152027f, b5 = -0.5f * 1.061405429f;
  constexpr float kE = -0.72134752044448170f;                 // -log2(e) / 2
  float2 a = make_float2(fabsf(g.x), fabsf(g.y));
  // the tail term is 0 beyond |g| ~ 13; the clamp keeps inf * 0 out of it
  const float2 ac = make_float2(fminf(a.x, 64.f), fminf(a.y, 64.f));
  const float2 den = f2fma(ac, f2s(kP), f2s(1.f));
  const float2 t = make_float2(rcp_approx(den.x), rcp_approx(den.y));
  float2 q = f2fma(t, f2s(b5), f2s(b4));
  q = f2fma(t, q, f2s(b3));
  q = f2fma(t, q, f2s(b2));
  q = f2fma(t, q, f2s(b1));
  q = f2mul(t, q);                                            // -0.5 P(t)
  const float2 w = f2mul(f2mul(ac, ac), f2s(kE));
  const float2 e = make_float2(ex2_approx(w.x), ex2_approx(w.y));
  const float2 m = f2mul(f2mul(ac, e), q);                    // -0.5 |g| P(t) e^{-g^2/2}
  return f2fma(f2add(g, a), f2s(0.5f), m);
}

// 2-d mapping, no integer division: blockIdx.x picks a 8*blockDim-wide column
// slice of the row, each thread walks rows grid-stride (kGegluVec rows per
// round, all loads issued first, kept as raw registers until consumed).
// 32-bit offsets: the host checks rows * 2f < 2^31.
template <typename T>
__global__ void __launch_bounds__(128)
geglu_kernel(const T* __restrict__ proj, T* __restrict__ out, int rows, int f) {
  pdl_wait();
  const int c = (blockIdx.x * blockDim.x + threadIdx.x) * 8;
  if (c >= f) return;
  const T* src = proj + c;
  T* dst = out + c;
  const int rstride = gridDim.y;
  for (int m0 = blockIdx.y; m0 < rows; m0 += rstride * kGegluVec) {
    Raw8<T> h[kGegluVec], g[kGegluVec];
#pragma unroll
    for (int u = 0; u < kGegluVec; ++u) {
      const int m = m0 + u * rstride;
      if (m < rows) {
        h[u] = load_raw<T>(src + (unsigned)m * (unsigned)(2 * f));
        g[u] = load_raw<T>(src + (unsigned)m * (unsigned)(2 * f) + f);
      }
    }
#pragma unroll
    for (int u = 0; u < kGegluVec; ++u) {
      const int m = m0 + u * rstride;
      if (m < rows) {
        Raw8<T> o;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float2 gv = get_pair<T>(g[u], i);
          float2 ge;
          if constexpr (sizeof(T) == 4) {   // fp32 parity mode: libdevice erff (torch's exact GELU)
            ge = make_float2(0.5f * gv.x * (1.f + erff(gv.x * 0.70710678118654752f)),
                             0.5f * gv.y * (1.f + erff(gv.y * 0.70710678118654752f)));
          } else {
            ge = gelu2(gv);
          }
          set_pair<T>(o, i, f2mul(get_pair<T>(h[u], i), ge));
        }
        store_raw<T>(dst + (unsigned)m * (unsigned)f, o);
      }
    }
  }
}

// ---- K5' the FF projection GEMM with GEGLU in its epilogue (tcgen05) -------
// out[m, j] = (x W_v^T + b_v)[m, j] * gelu((x W_g^T + b_g)[m, j]),
// W = [W_v; W_g] (2F x K, the diffusers GEGLU proj weight as stored).  The
// library path writes the 2F-wide projection and K5 reads it back (a 64²-level
// call: 84 MB out + 84 MB in + 42 MB out); here each 128 x 256 accumulator
// tile holds 128 value columns AND the matching 128 gate columns (two TMA
// boxes of W per K step: rows [128 n, 128 n + 128) and [F + 128 n, ...)), so
// the epilogue gates in registers and only the F-wide result is written.
// Persistent, warp-specialised: warp 0 TMA producer (4-stage ring of A 128 x
// 64 + B 256 x 64 bf16, 128-B swizzled), warp 1 the tcgen05 issuer
// (M128 N256 K16, fp32 in TMEM, two 256-column accumulators), warps 2-9 the
// epilogue (TMEM lane quadrant = warp % 4, two warps per quadrant splitting
// the 128 output columns; one row per thread; the tile's biases staged in
// shared memory).
constexpr int kFgBM = 128, kFgBN = 256, kFgBK = 64, kFgStages = 4;
constexpr int kFgEpiWarps = 8;                                   // two per TMEM lane quadrant
constexpr int kFgThreads = 64 + 32 * kFgEpiWarps;
constexpr int kFgStageBytes = kFgBM * 128 + kFgBN * 128;          // 48 KB
constexpr int kFgSmem = 1024 + kFgStages * kFgStageBytes + 256 + 2 * 256 * 4;

__global__ void __launch_bounds__(kFgThreads, 1)
ff_geglu_kernel(const __grid_constant__ CUtensorMap amap, const __grid_constant__ CUtensorMap bmap,
                const float* __restrict__ bias, __nv_bfloat16* __restrict__ out, int M, int K, int F, int tiles_n,
                int total) {
  extern __shared__ __align__(1024) uint8_t fg_smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(fg_smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kFgStages * kFgStageBytes);   // full[S] empty[S] tfull[2] tempty[2]
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 2 * kFgStages + 4);
  __shared__ float sbias[2 * 256];   // the tile's value | gate biases, per accumulator (static: plain LDS)
  constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kFgBN >> 3) << 17) |
                              ((uint32_t)(kFgBM >> 4) << 24);       // f32 accum, bf16 A/B, K-major, 128 x 256
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  auto full = [&](int s) { return smem_u32(bars + s); };
  auto empty = [&](int s) { return smem_u32(bars + kFgStages + s); };
  auto tfull = [&](int b) { return smem_u32(bars + 2 * kFgStages + b); };
  auto tempty = [&](int b) { return smem_u32(bars + 2 * kFgStages + 2 + b); };
  if (tid == 0) {
    prefetch_map(&amap);
    prefetch_map(&bmap);
    for (int s = 0; s < kFgStages; ++s) {
      mbar_init(full(s), 1);
      mbar_init(empty(s), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(tfull(b), 1);
      mbar_init(tempty(b), kFgEpiWarps);
    }
    mbar_fence_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  pdl_wait();
  const int nk = K / kFgBK;
  if (warp == 0) {
    if (lane == 0) {                                                // ---- TMA producer
      const uint64_t pol_a = policy_evict_first(), pol_b = policy_evict_last();
      int s = 0, round = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        const int tm = t / tiles_n, tn = t - tm * tiles_n;
        for (int k = 0; k < nk; ++k) {
          if (round > 0) mbar_wait(empty(s), (round - 1) & 1);
          uint8_t* st = smem + s * kFgStageBytes;
          mbar_expect_tx(full(s), kFgStageBytes);
          tma_load_2d(smem_u32(st), &amap, k * kFgBK, tm * kFgBM, full(s), pol_a);
          tma_load_2d(smem_u32(st + kFgBM * 128), &bmap, k * kFgBK, tn * 128, full(s), pol_b);
          tma_load_2d(smem_u32(st + kFgBM * 128 + 128 * 128), &bmap, k * kFgBK, F + tn * 128, full(s), pol_b);
          if (++s == kFgStages) { s = 0; ++round; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {                                                // ---- tcgen05 issuer
      int s = 0, round = 0, tl = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x, ++tl) {
        const int buf = tl & 1, use = tl >> 1;
        if (use > 0) mbar_wait(tempty(buf), (use - 1) & 1);
        tc_fence_after();
        const uint32_t d = tmem + (uint32_t)(buf * kFgBN);
        for (int k = 0; k < nk; ++k) {
          mbar_wait(full(s), round & 1);
          tc_fence_after();
          const uint32_t a = smem_u32(smem + s * kFgStageBytes), b = a + kFgBM * 128;
#pragma unroll
          for (int ks = 0; ks < 4; ++ks)
            tc_mma(d, sw128_desc(a + ks * 32), sw128_desc(b + ks * 32), kIdesc, (k | ks) ? 1u : 0u);
          tc_commit(empty(s));                                      // the stage is free once these MMAs are done
          if (++s == kFgStages) { s = 0; ++round; }
        }
        tc_commit(tfull(buf));
      }
    }
  } else {                                                          // ---- epilogue: warps 2..9
    const int q = warp & 3;                                         // TMEM lane quadrant this warp may read
    const int half = (warp - 2) >> 2;                               // which 64 of the 128 output columns
    const int r = q * 32 + lane;
    int tl = 0;
    const int et = tid - 64;                                        // 0..255 over the epilogue warps
    for (int t = blockIdx.x; t < total; t += gridDim.x, ++tl) {
      const int buf = tl & 1, use = tl >> 1;
      const int tm = t / tiles_n, tn = t - tm * tiles_n;
      // the tile's 128 value + 128 gate biases into shared memory while its MMAs run
      float* tb = sbias + buf * 256;
      if (bias != nullptr) tb[et] = __ldg(bias + (et < 128 ? tn * 128 + et : F + tn * 128 + et - 128));
      named_bar(1, 32 * kFgEpiWarps);
      mbar_wait(tfull(buf), use & 1);
      tc_fence_after();
      const uint32_t base = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(buf * kFgBN);
      const int row = tm * kFgBM + r;
      const int col0 = tn * 128;
      __nv_bfloat16* orow = out + (size_t)row * F + col0;
#pragma unroll 1
      for (int c0 = half * 64; c0 < half * 64 + 64; c0 += 32) {
        float v[32], g[32];
        tc_ld32(base + c0, v);
        tc_ld32(base + 128 + c0, g);
        if (row < M) {
          uint32_t pk[16];
#pragma unroll
          for (int j = 0; j < 32; j += 2) {
            float2 hv = make_float2(v[j], v[j + 1]), gv = make_float2(g[j], g[j + 1]);
            if (bias != nullptr) {
              hv = f2add(hv, *reinterpret_cast<const float2*>(tb + c0 + j));
              gv = f2add(gv, *reinterpret_cast<const float2*>(tb + 128 + c0 + j));
            }
            const float2 o = f2mul(hv, gelu2(gv));
            __nv_bfloat162 h2 = __floats2bfloat162_rn(o.x, o.y);
            pk[j >> 1] = *reinterpret_cast<uint32_t*>(&h2);
          }
#pragma unroll
          for (int i = 0; i < 4; ++i)
            *reinterpret_cast<uint4*>(orow + c0 + 8 * i) = make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty(buf));
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

// CTA-pair form (cta_group::2): one 256-row x 256-column accumulator tile per
// pair — each CTA TMA-loads its own 128 rows of x and ONE of the two W boxes
// (the leader the value rows, the follower the gate rows: the MMA's N = 256 is
// the leader's 128 B rows then the follower's), so a K step moves 32 KB per
// CTA instead of 48 and six stages fit; the leader issues M256 MMAs, every
// CTA's TMEM receives its 128 rows x [value | gate] and runs the same
// epilogue.  Loads of both CTAs complete on the leader's barriers; commits
// multicast to both.
constexpr int kFpStages = 6;
constexpr int kFpStageBytes = 128 * 128 + 128 * 128;              // A half + B half: 32 KB
constexpr int kFpSmem = 1024 + kFpStages * kFpStageBytes + 512 + 2 * 256 * 4;

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kFgThreads, 1)
ff_geglu_pair_kernel(const __grid_constant__ CUtensorMap amap, const __grid_constant__ CUtensorMap bmap,
                     const float* __restrict__ bias, __nv_bfloat16* __restrict__ out, int M, int K, int F,
                     int tiles_n, int total) {
  extern __shared__ __align__(1024) uint8_t fp_smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(fp_smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kFpStages * kFpStageBytes);   // full[S] empty[S] tfull[2] tempty[2]
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 2 * kFpStages + 4);
  __shared__ float sbias[2 * 256];   // the tile's value | gate biases, per accumulator (static: plain LDS)
  constexpr uint32_t kIdesc2 = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(256 >> 3) << 17) |
                               ((uint32_t)(256 >> 4) << 24);       // f32 accum, bf16, K-major, M256 x N256
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t cta = cluster_ctarank();
  const bool leader = cta == 0;
  const int cid = (int)cluster_idx(), ncl = (int)cluster_count();
  auto full = [&](int s) { return smem_u32(bars + s); };
  auto empty = [&](int s) { return smem_u32(bars + kFpStages + s); };
  auto tfull = [&](int b) { return smem_u32(bars + 2 * kFpStages + b); };
  auto tempty = [&](int b) { return smem_u32(bars + 2 * kFpStages + 2 + b); };
  if (tid == 0) {
    prefetch_map(&amap);
    prefetch_map(&bmap);
    for (int s = 0; s < kFpStages; ++s) {
      mbar_init(full(s), 1);
      mbar_init(empty(s), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(tfull(b), 1);
      mbar_init(tempty(b), 2 * kFgEpiWarps);                        // both CTAs' epilogue warps
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  pdl_wait();
  const int nk = K / kFgBK;
  if (warp == 0) {
    if (lane == 0) {                                                // ---- TMA producer (both CTAs)
      const uint64_t pol_a = policy_evict_first(), pol_b = policy_evict_last();
      int s = 0, round = 0;
      for (int t = cid; t < total; t += ncl) {
        const int tm = t / tiles_n, tn = t - tm * tiles_n;
        for (int k = 0; k < nk; ++k) {
          if (round > 0) mbar_wait(empty(s), (round - 1) & 1);
          uint8_t* st = smem + s * kFpStageBytes;
          if (leader) mbar_expect_tx(full(s), 2 * kFpStageBytes);
          const uint32_t lb = mapa_shared(full(s), 0);
          tma_load_2d_pair(smem_u32(st), &amap, k * kFgBK, tm * 256 + (int)cta * 128, lb, pol_a);
          tma_load_2d_pair(smem_u32(st + 128 * 128), &bmap, k * kFgBK, (int)cta * F + tn * 128, lb, pol_b);
          if (++s == kFpStages) { s = 0; ++round; }
        }
      }
      // drain: the leader's last multicast commits must land before this CTA exits
      for (int i = 0; i < kFpStages; ++i) {
        const int uses = round + (i < s ? 1 : 0);
        if (uses > 0) mbar_wait(empty(i), (uses - 1) & 1);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (leader && lane == 0) {                                      // ---- tcgen05 issuer (leader)
      int s = 0, round = 0, tl = 0;
      for (int t = cid; t < total; t += ncl, ++tl) {
        const int buf = tl & 1, use = tl >> 1;
        if (use > 0) mbar_wait(tempty(buf), (use - 1) & 1);
        tc_fence_after();
        const uint32_t d = tmem + (uint32_t)(buf * kFgBN);
        for (int k = 0; k < nk; ++k) {
          mbar_wait(full(s), round & 1);
          tc_fence_after();
          const uint32_t a = smem_u32(smem + s * kFpStageBytes), b = a + 128 * 128;
#pragma unroll
          for (int ks = 0; ks < 4; ++ks)
            tc_mma2(d, sw128_desc(a + ks * 32), sw128_desc(b + ks * 32), kIdesc2, (k | ks) ? 1u : 0u);
          tc_commit2(empty(s));
          if (++s == kFpStages) { s = 0; ++round; }
        }
        tc_commit2(tfull(buf));
      }
    }
    __syncwarp();
  } else {                                                          // ---- epilogue: warps 2..9 (each CTA)
    const int q = warp & 3;
    const int half = (warp - 2) >> 2;
    const int r = q * 32 + lane;
    const int et = tid - 64;
    int tl = 0;
    for (int t = cid; t < total; t += ncl, ++tl) {
      const int buf = tl & 1, use = tl >> 1;
      const int tm = t / tiles_n, tn = t - tm * tiles_n;
      float* tb = sbias + buf * 256;
      if (bias != nullptr) tb[et] = __ldg(bias + (et < 128 ? tn * 128 + et : F + tn * 128 + et - 128));
      named_bar(1, 32 * kFgEpiWarps);
      mbar_wait(tfull(buf), use & 1);
      tc_fence_after();
      const uint32_t base = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(buf * kFgBN);
      const int row = tm * 256 + (int)cta * 128 + r;
      const int col0 = tn * 128;
      __nv_bfloat16* orow = out + (size_t)row * F + col0;
#pragma unroll 1
      for (int c0 = half * 64; c0 < half * 64 + 64; c0 += 32) {
        float v[32], g[32];
        tc_ld32(base + c0, v);
        tc_ld32(base + 128 + c0, g);
        if (row < M) {
          uint32_t pk[16];
#pragma unroll
          for (int j = 0; j < 32; j += 2) {
            float2 hv = make_float2(v[j], v[j + 1]), gv = make_float2(g[j], g[j + 1]);
            if (bias != nullptr) {
              hv = f2add(hv, *reinterpret_cast<const float2*>(tb + c0 + j));
              gv = f2add(gv, *reinterpret_cast<const float2*>(tb + 128 + c0 + j));
            }
            const float2 o = f2mul(hv, gelu2(gv));
            __nv_bfloat162 h2 = __floats2bfloat162_rn(o.x, o.y);
            pk[j >> 1] = *reinterpret_cast<uint32_t*>(&h2);
          }
#pragma unroll
          for (int i = 0; i < 4; ++i)
            *reinterpret_cast<uint4*>(orow + c0 + 8 * i) = make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (leader) mbar_arrive(tempty(buf));
        else mbar_arrive_remote(mapa_shared(tempty(buf), 0));
      }
    }
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

// One warp per row, NV = vectors of 8 per lane (C <= 256 * NV).  Every load of
// the row (x, d) is issued before any is consumed; the rounded residual x + d
// is kept as raw T registers (it is stored in T, so nothing is lost) and both
// reductions and the output read it back — half the registers of an fp32 copy,
// so more rows are in flight per SM.  gamma / beta are re-read per row from L1.
template <typename T, int NV>
__global__ void __launch_bounds__(128)
add_layernorm_kernel(T* x, const T* __restrict__ d, T* __restrict__ y, const T* __restrict__ gamma,
                     const T* __restrict__ beta, int rows, int c, float eps) {
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int warps_total = gridDim.x * (blockDim.x >> 5);
  for (int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); row < rows; row += warps_total) {
    const size_t base = (size_t)row * c;
    Raw8<T> vq[NV], dq[NV];
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      const int col = (k * 32 + lane) * 8;
      if (col < c) {
        vq[k] = load_raw<T>(x + base + col);
        if (d != nullptr) dq[k] = load_raw<T>(d + base + col);
      }
    }
    float2 s = f2s(0.f);
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      const int col = (k * 32 + lane) * 8;
      if (col < c) {
        if (d != nullptr) {
          // the residual stream is stored in T: round once, normalise the stored value
#pragma unroll
          for (int i = 0; i < 4; ++i) set_pair<T>(vq[k], i, f2add(get_pair<T>(vq[k], i), get_pair<T>(dq[k], i)));
          store_raw<T>(x + base + col, vq[k]);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) s = f2add(s, get_pair<T>(vq[k], i));
      }
    }
    float sum = s.x + s.y;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    const float mean = sum / (float)c;
    const float2 nm = f2s(-mean);
    float2 q = f2s(0.f);
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      const int col = (k * 32 + lane) * 8;
      if (col < c) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float2 t = f2add(get_pair<T>(vq[k], i), nm);
          q = f2fma(t, t, q);
        }
      }
    }
    float sq = q.x + q.y;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
    // fp32 parity mode: an IEEE square root and division (rsqrtf is ~2 ulp)
    const float2 rstd = f2s(sizeof(T) == 4 ? 1.f / sqrtf(sq / (float)c + eps) : rsqrtf(sq / (float)c + eps));
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      const int col = (k * 32 + lane) * 8;
      if (col < c) {
        const Raw8<T> gq = load_raw<T>(gamma + col), bq = load_raw<T>(beta + col);
        Raw8<T> o;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float2 t = f2mul(f2add(get_pair<T>(vq[k], i), nm), rstd);
          set_pair<T>(o, i, f2fma(t, get_pair<T>(gq, i), get_pair<T>(bq, i)));
        }
        store_raw<T>(y + base + col, o);
      }
    }
  }
}

template <typename T>
int run_geglu(const void* proj, void* out, int64_t rows, int64_t f, cudaStream_t st) {
  if (rows * 2 * f >= (int64_t)INT32_MAX) return fail(SDB_EINVAL, "geglu: input must hold < 2^31 elements");
  const unsigned gx = (unsigned)((f / 8 + 127) / 128);
  // ~16 CTAs of 128 threads per SM in flight overall
  const int64_t want_y = std::max<int64_t>(1, (int64_t)kNumSMs * 16 / gx);
  const unsigned gy = (unsigned)std::min<int64_t>(std::min<int64_t>(want_y, (rows + kGegluVec - 1) / kGegluVec), 65535);
  launch_k(geglu_kernel<T>, dim3(gx, std::max(gy, 1u)), 128, 0, st, static_cast<const T*>(proj), static_cast<T*>(out),
                                                               (int)rows, (int)f);
  return check_launch("geglu_kernel");
}

template <typename T>
int run_add_ln(void* x, const void* d, void* y, const void* gamma, const void* beta, int64_t rows, int64_t c,
               float eps, cudaStream_t st) {
  if (rows >= (int64_t)INT32_MAX) return fail(SDB_EINVAL, "add_layernorm: too many rows");
  // 4 warps per 128-thread CTA, each warp walks rows grid-stride; ~8 CTAs per SM
  const unsigned grid = (unsigned)std::min<int64_t>((rows + 3) / 4, (int64_t)kNumSMs * 8);
  T* xp = static_cast<T*>(x);
  const T* dp = static_cast<const T*>(d);
  T* yp = static_cast<T*>(y);
  const T* gp = static_cast<const T*>(gamma);
  const T* bp = static_cast<const T*>(beta);
  const int nv = (int)((c / 8 + 31) / 32);
  switch (nv) {
    case 1: launch_k(add_layernorm_kernel<T, 1>, grid, 128, 0, st, xp, dp, yp, gp, bp, rows, c, eps); break;
    case 2: launch_k(add_layernorm_kernel<T, 2>, grid, 128, 0, st, xp, dp, yp, gp, bp, rows, c, eps); break;
    case 3: launch_k(add_layernorm_kernel<T, 3>, grid, 128, 0, st, xp, dp, yp, gp, bp, rows, c, eps); break;
    case 4: launch_k(add_layernorm_kernel<T, 4>, grid, 128, 0, st, xp, dp, yp, gp, bp, rows, c, eps); break;
    case 5: launch_k(add_layernorm_kernel<T, 5>, grid, 128, 0, st, xp, dp, yp, gp, bp, rows, c, eps); break;
    case 6: launch_k(add_layernorm_kernel<T, 6>, grid, 128, 0, st, xp, dp, yp, gp, bp, rows, c, eps); break;
    case 7: launch_k(add_layernorm_kernel<T, 7>, grid, 128, 0, st, xp, dp, yp, gp, bp, rows, c, eps); break;
    case 8: launch_k(add_layernorm_kernel<T, 8>, grid, 128, 0, st, xp, dp, yp, gp, bp, rows, c, eps); break;
    case 9: launch_k(add_layernorm_kernel<T, 9>, grid, 128, 0, st, xp, dp, yp, gp, bp, rows, c, eps); break;
    case 10: launch_k(add_layernorm_kernel<T, 10>, grid, 128, 0, st, xp, dp, yp, gp, bp, rows, c, eps); break;
    default: return fail(SDB_EINVAL, "add_layernorm: channels must be <= 2560");
  }
  return check_launch("add_layernorm_kernel");
}

// ---- batched copy (unpatch by restoring the pristine weights) ---------------
// Every tensor of a list copied by ONE launch: tensor t's 16-B vectors are cut
// into kCopyChunk-vector chunks; chunk_prefix[t] is the first chunk of tensor
// t (exclusive prefix, n + 1 entries), so a CTA finds its tensor with one
// binary search per chunk and streams the chunk with 16-B loads / stores,
// kCopyUnroll in flight per thread.  The reference's unmerge restores W by
// subtracting (lora.py:107-114); a serving copy can restore it exactly.
constexpr int kCopyThreads = 256, kCopyUnroll = 4;
constexpr int64_t kCopyChunk = (int64_t)kCopyThreads * kCopyUnroll * 8;   // vectors per chunk (128 KB)

struct CopyTable {
  const uint4* const* src;
  uint4* const* dst;
  const int64_t* nvec;          // 16-B vectors per tensor
  const int64_t* chunk_prefix;  // n + 1
  int n;
};

__global__ void __launch_bounds__(kCopyThreads) batched_copy_kernel(CopyTable t) {
  pdl_wait();
  const int64_t chunks = t.chunk_prefix[t.n];
  for (int64_t ch = blockIdx.x; ch < chunks; ch += gridDim.x) {
    int lo = 0, hi = t.n - 1;                   // last tensor whose first chunk <= ch
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (t.chunk_prefix[mid] <= ch) lo = mid; else hi = mid - 1;
    }
    const int64_t v0 = (ch - t.chunk_prefix[lo]) * kCopyChunk;
    const int64_t v1 = min(t.nvec[lo], v0 + kCopyChunk);
    const uint4* __restrict__ s = t.src[lo];
    uint4* __restrict__ d = t.dst[lo];
    for (int64_t v = v0 + threadIdx.x; v < v1; v += (int64_t)kCopyThreads * kCopyUnroll) {
      uint4 q[kCopyUnroll];
#pragma unroll
      for (int u = 0; u < kCopyUnroll; ++u)
        if (v + u * kCopyThreads < v1) q[u] = __ldcs(s + v + u * kCopyThreads);   // streamed once
#pragma unroll
      for (int u = 0; u < kCopyUnroll; ++u)
        if (v + u * kCopyThreads < v1) __stcs(d + v + u * kCopyThreads, q[u]);
    }
  }
}

}  // namespace

// K10 nearest 2x upsample, NHWC: y[n, 2i+a, 2j+b, :] = x[n, i, j, :].  One
// 16-B vector (8 channels) in, four 16-B vectors out; the library NHWC
// interpolate kernel took 59 / 116 us for SDXL's [2,1280,32,32] /
// [2,640,64,64] (scripts/upsample_probe.py), i.e. ~5% of the HBM rate.
__global__ void __launch_bounds__(256)
upsample2x_kernel(const uint4* __restrict__ x, uint4* __restrict__ y, int64_t total, int w, int cv) {
  pdl_wait();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i % cv);
    const int64_t p = i / cv;                   // input pixel (n, i, j), row-major
    const int j = (int)(p % w);
    const int64_t ni = p / w;                   // n * h + i
    const uint4 v = x[i];
    const int64_t o = ((ni * 2) * (2 * w) + 2 * j) * cv + c;   // (n, 2i, 2j)
    y[o] = v;
    y[o + cv] = v;
    y[o + 2 * w * cv] = v;
    y[o + 2 * w * cv + cv] = v;
  }
}

// K5': out[M, F] = GEGLU(x[M, K] W[2F, K]^T + bias[2F]) in one tcgen05 GEMM.
// bf16 only; K % 64 == 0, F % 128 == 0, row strides dense (x: K, W: K, out: F).
int ff_geglu(const void* x, const void* w, const float* bias, void* out, int64_t m, int64_t k, int64_t f,
             cudaStream_t st) {
  if (m <= 0 || k <= 0 || f <= 0) return fail(SDB_EINVAL, "ff_geglu: empty shape");
  if (k % kFgBK != 0 || f % 128 != 0) return fail(SDB_EUNSUP, "ff_geglu: K % 64 and F % 128 must be 0");
  if (m * f >= ((int64_t)1 << 31) || m >= ((int64_t)1 << 31)) return fail(SDB_EINVAL, "ff_geglu: too large");
  if (((uintptr_t)x | (uintptr_t)w | (uintptr_t)out | (uintptr_t)bias) & 15)
    return fail(SDB_EINVAL, "ff_geglu: pointers must be 16-byte aligned");
  EncodeTiledFn enc = encode_fn();
  if (!enc) return fail(SDB_ECUDA, "cuTensorMapEncodeTiled unavailable");
  CUtensorMap am, bm;
  const cuuint32_t es[2] = {1, 1};
  {
    const cuuint64_t dims[2] = {(cuuint64_t)k, (cuuint64_t)m};
    const cuuint64_t strides[1] = {(cuuint64_t)k * 2};
    const cuuint32_t box[2] = {(cuuint32_t)kFgBK, (cuuint32_t)kFgBM};
    if (enc(&am, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(x), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return fail(SDB_EINVAL, "ff_geglu: x tensor map");
  }
  {
    const cuuint64_t dims[2] = {(cuuint64_t)k, (cuuint64_t)(2 * f)};
    const cuuint64_t strides[1] = {(cuuint64_t)k * 2};
    const cuuint32_t box[2] = {(cuuint32_t)kFgBK, 128u};
    if (enc(&bm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(w), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return fail(SDB_EINVAL, "ff_geglu: weight tensor map");
  }
  const int tiles_n = (int)(f / 128);
  static int pair = -1;   // SDB_FF_PAIR=0: the single-CTA form (probe knob)
  if (pair < 0) {
    const char* e = getenv("SDB_FF_PAIR");
    pair = (e != nullptr && e[0] == '0') ? 0 : 1;
  }
  if (pair) {
    const int tiles_m = (int)((m + 255) / 256);
    const int total = tiles_m * tiles_n;
    static bool pattr = false;
    if (!pattr) {
      cudaFuncSetAttribute(ff_geglu_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kFpSmem);
      pattr = true;
    }
    const int clusters = std::min(total, kNumSMs / 2);
    launch_k(ff_geglu_pair_kernel, dim3((unsigned)(2 * clusters)), kFgThreads, kFpSmem, st, am, bm, bias,
             static_cast<__nv_bfloat16*>(out), (int)m, (int)k, (int)f, tiles_n, total);
    return check_launch("ff_geglu_pair_kernel");
  }
  const int tiles_m = (int)((m + kFgBM - 1) / kFgBM);
  const int total = tiles_m * tiles_n;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(ff_geglu_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kFgSmem);
    attr = true;
  }
  const int grid = std::min(total, kNumSMs);
  launch_k(ff_geglu_kernel, dim3((unsigned)grid), kFgThreads, kFgSmem, st, am, bm, bias,
           static_cast<__nv_bfloat16*>(out), (int)m, (int)k, (int)f, tiles_n, total);
  return check_launch("ff_geglu_kernel");
}

int geglu(const void* proj, void* out, int64_t rows, int64_t f, int dtype, cudaStream_t st) {
  if (rows <= 0 || f <= 0 || f % 8 != 0) return fail(SDB_EINVAL, "geglu: width must be a positive multiple of 8");
  if ((reinterpret_cast<uintptr_t>(proj) | reinterpret_cast<uintptr_t>(out)) & 15)
    return fail(SDB_EINVAL, "geglu: pointers must be 16-byte aligned");
  switch (dtype) {
    case SDB_BF16: return run_geglu<__nv_bfloat16>(proj, out, rows, f, st);
    case SDB_F16: return run_geglu<__half>(proj, out, rows, f, st);
    case SDB_F32: return run_geglu<float>(proj, out, rows, f, st);
    default: return fail(SDB_EUNSUP, "geglu: unsupported dtype");
  }
}

int add_layernorm(void* x, const void* d, void* y, const void* gamma, const void* beta, int64_t rows, int64_t c,
                  float eps, int dtype, cudaStream_t st) {
  if (rows <= 0 || c <= 0 || c % 8 != 0) return fail(SDB_EINVAL, "add_layernorm: channels must be a multiple of 8");
  if (!x || !y || !gamma || !beta) return fail(SDB_EINVAL, "add_layernorm: NULL pointer");
  if ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(d) | reinterpret_cast<uintptr_t>(y) |
       reinterpret_cast<uintptr_t>(gamma) | reinterpret_cast<uintptr_t>(beta)) & 15)
    return fail(SDB_EINVAL, "add_layernorm: pointers must be 16-byte aligned");
  switch (dtype) {
    case SDB_BF16: return run_add_ln<__nv_bfloat16>(x, d, y, gamma, beta, rows, c, eps, st);
    case SDB_F16: return run_add_ln<__half>(x, d, y, gamma, beta, rows, c, eps, st);
    case SDB_F32: return run_add_ln<float>(x, d, y, gamma, beta, rows, c, eps, st);
    default: return fail(SDB_EUNSUP, "add_layernorm: unsupported dtype");
  }
}

int upsample2x(const void* x, void* y, int64_t n, int64_t h, int64_t w, int64_t c, int elem_bytes, cudaStream_t st) {
  if (n <= 0 || h <= 0 || w <= 0 || c <= 0) return fail(SDB_EINVAL, "upsample2x: empty shape");
  if ((c * elem_bytes) % 16 != 0) return fail(SDB_EINVAL, "upsample2x: C * element size must be a multiple of 16");
  if (((uintptr_t)x | (uintptr_t)y) & 15) return fail(SDB_EINVAL, "upsample2x: pointers must be 16-byte aligned");
  if (w > INT32_MAX / 2) return fail(SDB_EINVAL, "upsample2x: too wide");
  const int cv = (int)(c * elem_bytes / 16);
  const int64_t total = n * h * w * cv;
  const int64_t grid = std::min<int64_t>((total + 255) / 256, (int64_t)kNumSMs * 8);
  launch_k(upsample2x_kernel, (unsigned)grid, 256, 0, st, static_cast<const uint4*>(x), static_cast<uint4*>(y), total,
                                                    (int)w, cv);
  return check_launch("upsample2x_kernel");
}

int batched_copy(const void* const* src_dev, void* const* dst_dev, const int64_t* nvec_dev,
                 const int64_t* chunk_prefix_dev, int n, int64_t total_chunks, cudaStream_t st) {
  if (n <= 0 || total_chunks <= 0) return SDB_OK;
  CopyTable t{reinterpret_cast<const uint4* const*>(src_dev), reinterpret_cast<uint4* const*>(dst_dev), nvec_dev,
              chunk_prefix_dev, n};
  const int grid = (int)std::min<int64_t>(total_chunks, 8 * kNumSMs);
  launch_k(batched_copy_kernel, grid, kCopyThreads, 0, st, t);
  return check_launch("batched_copy_kernel");
}

int64_t batched_copy_chunk_vectors() { return kCopyChunk; }

}  // namespace sdb
