// cross_attn.cu — K7: cross-attention against a short, step-invariant text
// context (77 tokens for SD1.5/SDXL), one pass over the queries.
//
//   o[n, i, h*d:(h+1)*d] = softmax(q_h[i] . k_h^T / sqrt(d)) v_h
//   q: [N, Lq, C] (row stride ldq), kv: [N, Lk, 2C] = K|V (row stride ldkv,
//   V at column offset voff), o: [N, Lq, C] (row stride ldo), C = H * d.
//
// With Lk <= 128 the whole K_h / V_h of a head fits in shared memory and a
// query row's scores fit in registers, so there is no online softmax and no
// K/V loop: each CTA stages K_h, V_h once (<= 2 x 128 x 168 x 2 B) and its 8
// warps each take 16 queries through S = Q K^T (m16n8k16 bf16 MMA, fp32
// accumulate), an exact in-register softmax (quad shuffles), P -> bf16 and
// O = P V.  Per query the kernel reads q once and writes o once — the
// algorithmic minimum (the SDXL cross-attention moves 2 x 10.5 MB
// per 64x64-level call and does ~1.6 GFLOP, far below any tensor-pipe limit;
// the library flash kernel spent ~15 us on it, HBM needs ~3.3 us).  The
// reference has no attention at all (addonsim is a latency model); this
// kernel is part of the UNet backbone the north_star's denoising loop runs.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"

namespace sdb {
namespace {

constexpr int kWarps = 4;
constexpr int kThreads = kWarps * 32;
constexpr int kQRows = 16;   // queries per warp tile (MMA M)
constexpr int kSlots = 2;    // per-warp query-tile ring: tile i + 1 loads while tile i computes
constexpr int kTargetWarps = 148 * 12;   // warps to aim for: ~3 tiles per warp at SDXL's 64x64 level (measured best)

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void ldsm_x4(uint32_t a, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(a));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t a, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(a));
}
// 16-B global -> shared async copy; src_bytes = 0 zero-fills (padding rows / columns)
__device__ __forceinline__ void cp_async16(void* dst, const void* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_addr(dst)), "l"(src), "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <typename T>
__device__ __forceinline__ void mma16816(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1);
template <>
__device__ __forceinline__ void mma16816<__nv_bfloat16>(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                                        uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
template <>
__device__ __forceinline__ void mma16816<__half>(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                                 uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
// 2^x on the SFU without the accurate-path range fix-up (inputs are <= 0 and
// -inf for masked keys: ex2.approx.ftz gives 0 there, flushes denormals to 0)
__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float fast_rcp(float x) {   // row sums are >= 1 (the max term is 2^0)
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
template <typename T> __device__ __forceinline__ uint32_t pack2(float lo, float hi);
template <> __device__ __forceinline__ uint32_t pack2<__nv_bfloat16>(float lo, float hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}
template <> __device__ __forceinline__ uint32_t pack2<__half>(float lo, float hi) {
  __half2 h = __floats2half2_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}

// DP: head dim padded to a multiple of 16 (MMA K of S = Q K^T and the row
// count of O's N chunks); NKP: keys padded to a multiple of 16 (MMA K of P V).
// Shared-memory operands are addressed as one per-lane base + compile-time
// offsets, and B fragments come two MMA columns per ldmatrix.x4, so the
// unrolled body is almost only LDSM / HMMA / the softmax arithmetic.
template <typename T, int DP, int NKP>
__global__ void __launch_bounds__(kThreads)
cross_attn_kernel(const T* __restrict__ q, int64_t ldq, const T* __restrict__ kv, int64_t ldkv, int64_t voff,
                  T* __restrict__ o, int64_t ldo, int lq, int lk, int d, float scale_log2, int tpw) {
  constexpr int LDS = DP + 8;                     // smem row pitch (elements): 16 B skew, no ldmatrix conflicts
  constexpr int NC = NKP / 8;                     // key chunks of 8 (S columns)
  constexpr int DC = DP / 8;                      // head-dim chunks of 8 (O columns)
  constexpr int SLOT = kQRows * LDS;              // one query tile (elements)
  static_assert(NC % 2 == 0 && DC % 2 == 0, "chunk pairs");
  extern __shared__ __align__(16) uint8_t xa_smem[];
  T* sK = reinterpret_cast<T*>(xa_smem);
  T* sV = sK + NKP * LDS;
  T* sQ = sV + NKP * LDS + (threadIdx.x >> 5) * kSlots * SLOT;   // this warp's tile ring

  const int h = blockIdx.y, n = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int dv = d >> 3;                          // 16-B vectors per head row
  const T* kbase = kv + (int64_t)n * lk * ldkv + (int64_t)h * d;
  const T* qbase = q + (int64_t)n * lq * ldq + (int64_t)h * d;
  T* obase = o + (int64_t)n * lq * ldo + (int64_t)h * d;
  const int first = (blockIdx.x * kWarps + warp) * tpw * kQRows;   // this warp's first query
  const int ntiles = max(0, min(tpw, (lq - first + kQRows - 1) / kQRows));

  // async copy of query tile i into ring slot i % kSlots (rows >= lq, cols >= d zero-filled)
  // (a lane's (row, chunk) pattern is fixed: kQRows * DC / 32 = DC / 2 copies)
  auto load_tile = [&](int i) {
    T* sq = sQ + (i % kSlots) * SLOT;
    const int q0 = first + i * kQRows;
#pragma unroll
    for (int k = 0; k < DC / 2; ++k) {
      const int e = lane + 32 * k, r = e / DC, c = e % DC;
      const bool ok = q0 + r < lq && c < dv;
      cp_async16(sq + r * LDS + c * 8, qbase + (ok ? (uint32_t)(q0 + r) * (uint32_t)ldq + c * 8 : 0), ok ? 16 : 0);
    }
  };
  // ---- K_h, V_h (group 0) and the first query tile (group 1) in flight together
  for (int i = threadIdx.x; i < NKP * DC; i += kThreads) {
    const int r = i / DC, c = i % DC;
    const bool ok = r < lk && c < dv;
    const T* src = kbase + (ok ? (int64_t)r * ldkv + c * 8 : 0);
    cp_async16(sK + r * LDS + c * 8, src, ok ? 16 : 0);
    cp_async16(sV + r * LDS + c * 8, src + (ok ? voff : 0), ok ? 16 : 0);
  }
  cp_async_commit();
  if (ntiles > 0) load_tile(0);
  cp_async_commit();
  cp_async_wait<1>();
  __syncthreads();

  // per-lane ldmatrix bases (bytes); every fragment is base + a constant
  //   K (x4): lanes 0-7 / 8-15 -> key chunk j, d lo / hi; 16-23 / 24-31 -> chunk j + 1
  //   V (x4.trans): lanes 0-15 -> key rows, d chunk dn; 16-31 -> d chunk dn + 1
  //   Q (x4): lanes 0-15 -> rows, d lo; 16-31 -> rows, d hi
  const uint32_t kl = smem_addr(sK + (((lane >> 4) << 3) + (lane & 7)) * LDS + ((lane >> 3) & 1) * 8);
  const uint32_t vl = smem_addr(sV + (lane & 15) * LDS + (lane >> 4) * 8);
  const uint32_t ql = smem_addr(sQ + (lane & 15) * LDS + (lane >> 4) * 8);
  const int t = lane & 3, g = lane >> 2;

#pragma unroll 1
  for (int i = 0; i < ntiles; ++i) {
    // prefetch the next tile into the other slot, then wait for this one
    if (i + 1 < ntiles) load_tile(i + 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncwarp();
    const int q0 = first + i * kQRows;
    const uint32_t qa = ql + (i % kSlots) * (SLOT * 2);

    // ---- S = Q K^T ---------------------------------------------------------
    float s[NC][4];
#pragma unroll
    for (int j = 0; j < NC; ++j) s[j][0] = s[j][1] = s[j][2] = s[j][3] = 0.f;
#pragma unroll
    for (int kc = 0; kc < DP / 16; ++kc) {
      uint32_t a0, a1, a2, a3;
      ldsm_x4(qa + kc * 32, a0, a1, a2, a3);
#pragma unroll
      for (int j = 0; j < NC; j += 2) {
        uint32_t b0, b1, b2, b3;
        ldsm_x4(kl + (j * 8 * LDS + kc * 16) * 2, b0, b1, b2, b3);
        mma16816<T>(s[j], a0, a1, a2, a3, b0, b1);
        mma16816<T>(s[j + 1], a0, a1, a2, a3, b2, b3);
      }
    }
    // ---- exact softmax over the keys of rows g and g + 8 --------------------
    // (padded keys only exist in the chunks past lk / 8: warp-uniform test)
#pragma unroll
    for (int j = 0; j < NC; ++j) {
      if (j * 8 + 8 > lk) {
        const int k0 = j * 8 + 2 * t;
        if (k0 >= lk) s[j][0] = s[j][2] = -INFINITY;
        if (k0 + 1 >= lk) s[j][1] = s[j][3] = -INFINITY;
      }
    }
    float m0 = s[0][0], m1 = s[0][2];
#pragma unroll
    for (int j = 0; j < NC; ++j) {
      m0 = fmaxf(m0, fmaxf(s[j][0], s[j][1]));
      m1 = fmaxf(m1, fmaxf(s[j][2], s[j][3]));
    }
#pragma unroll
    for (int off = 1; off <= 2; off <<= 1) {
      m0 = fmaxf(m0, __shfl_xor_sync(0xffffffffu, m0, off));
      m1 = fmaxf(m1, __shfl_xor_sync(0xffffffffu, m1, off));
    }
    const float mb0 = m0 * scale_log2, mb1 = m1 * scale_log2;
    float l0 = 0.f, l1 = 0.f;
#pragma unroll
    for (int j = 0; j < NC; ++j) {
      s[j][0] = fast_exp2(fmaf(s[j][0], scale_log2, -mb0));
      s[j][1] = fast_exp2(fmaf(s[j][1], scale_log2, -mb0));
      s[j][2] = fast_exp2(fmaf(s[j][2], scale_log2, -mb1));
      s[j][3] = fast_exp2(fmaf(s[j][3], scale_log2, -mb1));
      l0 += s[j][0] + s[j][1];
      l1 += s[j][2] + s[j][3];
    }
#pragma unroll
    for (int off = 1; off <= 2; off <<= 1) {
      l0 += __shfl_xor_sync(0xffffffffu, l0, off);
      l1 += __shfl_xor_sync(0xffffffffu, l1, off);
    }
    // ---- O = P V (P's C fragments re-used as A fragments) -----------------
    float acc[DC][4];
#pragma unroll
    for (int j = 0; j < DC; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < NKP / 16; ++kk) {
      const uint32_t a0 = pack2<T>(s[2 * kk][0], s[2 * kk][1]);
      const uint32_t a1 = pack2<T>(s[2 * kk][2], s[2 * kk][3]);
      const uint32_t a2 = pack2<T>(s[2 * kk + 1][0], s[2 * kk + 1][1]);
      const uint32_t a3 = pack2<T>(s[2 * kk + 1][2], s[2 * kk + 1][3]);
#pragma unroll
      for (int dn = 0; dn < DC; dn += 2) {
        uint32_t b0, b1, b2, b3;
        ldsm_x4_t(vl + (kk * 16 * LDS + dn * 8) * 2, b0, b1, b2, b3);
        mma16816<T>(acc[dn], a0, a1, a2, a3, b0, b1);
        mma16816<T>(acc[dn + 1], a0, a1, a2, a3, b2, b3);
      }
    }
    // ---- normalise, stage through this tile's slot, 16-B stores ------------
    const float r0 = fast_rcp(l0), r1 = fast_rcp(l1);
    T* sq = sQ + (i % kSlots) * SLOT;
    __syncwarp();
#pragma unroll
    for (int dn = 0; dn < DC; ++dn) {
      *reinterpret_cast<uint32_t*>(sq + g * LDS + dn * 8 + 2 * t) = pack2<T>(acc[dn][0] * r0, acc[dn][1] * r0);
      *reinterpret_cast<uint32_t*>(sq + (g + 8) * LDS + dn * 8 + 2 * t) =
          pack2<T>(acc[dn][2] * r1, acc[dn][3] * r1);
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < DC / 2; ++k) {
      const int e = lane + 32 * k, r = e / DC, c = e % DC;
      if (q0 + r < lq && c < dv)
        *reinterpret_cast<uint4*>(obase + (uint32_t)(q0 + r) * (uint32_t)ldo + c * 8) =
            *reinterpret_cast<const uint4*>(sq + r * LDS + c * 8);
    }
    __syncwarp();   // the slot's reads are done before a later prefetch overwrites it
  }
  cp_async_wait<0>();
}

template <typename T, int DP, int NKP>
int launch(const void* q, int64_t ldq, const void* kv, int64_t ldkv, int64_t voff, void* o, int64_t ldo,
           int n, int lq, int lk, int heads, int d, float scale, cudaStream_t st) {
  // tiles per warp: enough warps for one resident wave, each walking several
  // tiles so its loads overlap its math (SDXL: 3 at the 64x64 level, 2 at 32x32)
  const int64_t tiles = (int64_t)n * heads * ((lq + kQRows - 1) / kQRows);
  const int tpw = (int)std::max<int64_t>(1, (tiles + kTargetWarps - 1) / kTargetWarps);
  const int cta_q = kWarps * kQRows * tpw;
  dim3 grid((unsigned)((lq + cta_q - 1) / cta_q), (unsigned)heads, (unsigned)n);
  const int smem = (2 * NKP + kWarps * kSlots * kQRows) * (DP + 8) * (int)sizeof(T);
  static bool attr = false;   // per instantiation
  if (!attr) {
    cudaFuncSetAttribute(cross_attn_kernel<T, DP, NKP>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  cross_attn_kernel<T, DP, NKP><<<grid, kThreads, smem, st>>>(
      static_cast<const T*>(q), ldq, static_cast<const T*>(kv), ldkv, voff, static_cast<T*>(o), ldo, lq, lk, d,
      scale * 1.4426950408889634f, tpw);
  return check_launch("cross_attn_kernel");
}

template <typename T, int NKP>
int by_dim(const void* q, int64_t ldq, const void* kv, int64_t ldkv, int64_t voff, void* o, int64_t ldo, int n,
           int lq, int lk, int heads, int d, float scale, cudaStream_t st) {
  if (d <= 16) return launch<T, 16, NKP>(q, ldq, kv, ldkv, voff, o, ldo, n, lq, lk, heads, d, scale, st);
  if (d <= 48) return launch<T, 48, NKP>(q, ldq, kv, ldkv, voff, o, ldo, n, lq, lk, heads, d, scale, st);
  if (d <= 64) return launch<T, 64, NKP>(q, ldq, kv, ldkv, voff, o, ldo, n, lq, lk, heads, d, scale, st);
  if (d <= 80) return launch<T, 80, NKP>(q, ldq, kv, ldkv, voff, o, ldo, n, lq, lk, heads, d, scale, st);
  return launch<T, 160, NKP>(q, ldq, kv, ldkv, voff, o, ldo, n, lq, lk, heads, d, scale, st);
}

template <typename T>
int by_keys(const void* q, int64_t ldq, const void* kv, int64_t ldkv, int64_t voff, void* o, int64_t ldo, int n,
            int lq, int lk, int heads, int d, float scale, cudaStream_t st) {
  if (lk <= 16) return by_dim<T, 16>(q, ldq, kv, ldkv, voff, o, ldo, n, lq, lk, heads, d, scale, st);
  if (lk <= 80) return by_dim<T, 80>(q, ldq, kv, ldkv, voff, o, ldo, n, lq, lk, heads, d, scale, st);
  return by_dim<T, 128>(q, ldq, kv, ldkv, voff, o, ldo, n, lq, lk, heads, d, scale, st);
}

}  // namespace

int cross_attention(const void* q, int64_t ldq, const void* kv, int64_t ldkv, int64_t voff, void* o, int64_t ldo,
                    int n, int lq, int lk, int heads, int d, float scale, int dtype, cudaStream_t st) {
  if (n <= 0 || lq < 0 || heads <= 0) return fail(SDB_EINVAL, "cross_attention: bad N / Lq / heads");
  if (lk < 1 || lk > 128) return fail(SDB_EUNSUP, "cross_attention: context length must be in [1, 128]");
  if (d < 8 || d > 160 || d % 8 != 0) return fail(SDB_EUNSUP, "cross_attention: head dim must be 8..160, % 8");
  if ((ldq | ldkv | ldo | voff) % 8 != 0) return fail(SDB_EINVAL, "cross_attention: strides must be multiples of 8");
  if ((int64_t)lq * std::max(ldq, ldo) >= ((int64_t)1 << 31))
    return fail(SDB_EINVAL, "cross_attention: lq * row stride must be < 2^31");
  if (((uintptr_t)q | (uintptr_t)kv | (uintptr_t)o) & 15)
    return fail(SDB_EINVAL, "cross_attention: pointers must be 16-byte aligned");
  if ((int64_t)heads * d > ldq || (int64_t)heads * d > ldo || voff + (int64_t)heads * d > ldkv)
    return fail(SDB_EINVAL, "cross_attention: heads * d exceeds a row stride");
  if (lq == 0) return SDB_OK;
  switch (dtype) {
    case SDB_BF16: return by_keys<__nv_bfloat16>(q, ldq, kv, ldkv, voff, o, ldo, n, lq, lk, heads, d, scale, st);
    default: return fail(SDB_EUNSUP, "cross_attention: bf16 only");
  }
}

}  // namespace sdb
