// gn_cluster.cu — K2, single-pass form: GroupNorm (+ SiLU) of an NHWC bf16
// feature map held ENTIRELY in the shared memory of a thread-block cluster.
//
// Same semantics as groupnorm_silu.cu (torch.nn.GroupNorm then SiLU; the
// fused GN+SiLU the reference models as addonsim/model.py:66-70): per
// (sample, group) mean and biased variance over C/G channels x H x W, eps
// inside the rsqrt, per-channel affine, optional per-(n, c) add before the
// norm (the ResNet time-embedding projection).
//
// The two-pass form reads the map twice (stats, then apply) in two launches
// and its cost at SDXL's sizes is launch ramps and dependent round trips, not
// bytes.  Here one launch reads the map ONCE and writes it once:
//
//   * the channels are cut into slabs of S = lcm(C/G, 8) channels (whole
//     groups, 16-B rows) and the pixels of one sample into `cs` equal runs
//     (cs <= 16, raised until the launch spans ~128 CTAs); a cluster of cs
//     1024-thread CTAs owns one (sample, slab) and each CTA TMA-loads its
//     run x slab box (<= 200 KB) into shared memory;
//   * pass 1 (sums) and pass 2 (centred squares: an exact two-pass variance)
//     run over shared memory; per-thread fp32 partials fold per column, then
//     per group in a fixed order; the cluster exchanges the cs per-CTA group
//     partials through distributed shared memory (each CTA reads its peers'
//     fp64 partials with ld.shared::cluster after a cluster barrier) and sums
//     them in rank order — deterministic, no atomics, no workspace;
//   * apply + SiLU in place in shared memory, TMA store.
//
// Eligible shapes (host plan below): bf16, C/G >= 8, S <= 256, a divisor cs
// of H*W with H*W/cs rows fitting the tile budget, and a map <= 6 MB — the
// only size class where it measured faster than the two-pass form (SDXL's
// 32x32-level sites: [2, 1280, 32, 32] 12.5 us vs 16.3 us).  Everything else
// runs the two-pass form.
#include <cuda.h>

#include <algorithm>
#include <numeric>

#include "common.cuh"
#include "ptx.cuh"
#include "tcgen05.cuh"

namespace sdb {

int g_gn_cluster_mode = 0;   // 0 auto, 1 force the two-pass form (tests / probes)

namespace {

constexpr int kGcThreads = 1024;
constexpr int kGcMaxCs = 16;
constexpr int kGcMaxGs = 32;                   // groups per slab
constexpr int kGcTargetCtas = 128;
// measured (scripts/gn_cluster_probe.py, CUDA-graph replays, inputs > L2):
// the cluster form wins only on small maps — [2,1280,32,32] 12.5 us vs 16.3
// two-pass; ties at 10.5 MB; loses from 15.7 MB up (49 us vs 24 at
// [2,320,128,128]: larger clusters co-schedule in two waves and each SM
// then walks 160 KB through three dependent phases with one CTA's warps)
constexpr int64_t kGcMaxBytes = 6 << 20;
constexpr int kGcTileMax = 200 * 1024;         // tile bytes per CTA
constexpr int kGcExtra = kGcThreads * 8 + 32 * 32 * 8 + 32 * 8 + 2 * kGcMaxGs * 8 + 2 * kGcMaxGs * 4 + 16;

__device__ __forceinline__ uint32_t cl_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cl_size() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cl_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
__device__ __forceinline__ void cl_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }
__device__ __forceinline__ double ld_peer_f64(uint32_t local_addr, uint32_t rank) {
  uint32_t a;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(local_addr), "r"(rank));
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ float silu_fast(float y) {   // ex2 on the MUFU, 1/(1+e) by Newton on the FMA pipe
  float e;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(fminf(-1.4426950408889634f * y, 126.f)));
  const float d = 1.f + e;
  float x = __int_as_float(0x7EF311C3 - __float_as_int(d));
  x = x * fmaf(-d, x, 2.f);
  return y * (x * fmaf(-d, x, 2.f));
}

template <bool SILU>
__global__ void __launch_bounds__(kGcThreads, 1)
gn_cluster_kernel(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap ymap,
                  const float* __restrict__ gamma, const float* __restrict__ beta,
                  const float* __restrict__ add_nc, int hw, int c, int cpg, int S, int rows, int br, float eps) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int tile_bytes = rows * S * 2;
  uint8_t* tile = smem;
  float2* part = reinterpret_cast<float2*>(smem + ((tile_bytes + 127) & ~127));
  float2* s1 = part + kGcThreads;                                       // [32][VC] column partials
  float2* colsum = s1 + 32 * 32;                                        // [VC]
  double* ex = reinterpret_cast<double*>(colsum + 32);                 // [2][kGcMaxGs] cluster-visible
  float* stat = reinterpret_cast<float*>(ex + 2 * kGcMaxGs);           // mean[kGcMaxGs] | rstd[kGcMaxGs]
  uint64_t* mbar = reinterpret_cast<uint64_t*>(stat + 2 * kGcMaxGs);
  const uint32_t rank = cl_rank(), cs = cl_size();
  const int n = blockIdx.z;
  const int c0 = blockIdx.y * S;
  const int gs = S / cpg;
  const int tid = threadIdx.x;
  const int row0 = n * hw + (int)rank * rows;
  const uint32_t bar = smem_u32(mbar);
  if (tid == 0) {
    prefetch_map(&xmap);
    prefetch_map(&ymap);
    mbar_init(bar, 1);
    mbar_fence_init();
  }
  __syncthreads();
  if (tid == 0) {
    mbar_expect_tx(bar, (uint32_t)tile_bytes);
    const uint64_t pol = policy_evict_first();
    for (int k = 0; k < rows; k += br) tma_load_2d(smem_u32(tile + (size_t)k * S * 2), &xmap, c0, row0 + k, bar, pol);
  }
  // this thread's fixed 8-channel column (overlaps the load)
  const int VC = S >> 3;
  const int rstep = kGcThreads / VC;
  const int j = tid % VC;
  const int rstart = tid / VC;
  const bool active = rstart < rstep;
  const int ch0 = j * 8;
  const int gA = ch0 / cpg;
  const int nA = min(8, (gA + 1) * cpg - ch0);        // leading elements in group gA, the rest in gA + 1
  float addv[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) addv[e] = add_nc != nullptr ? add_nc[(size_t)n * c + c0 + ch0 + e] : 0.f;
  mbar_wait(bar, 0);

  auto load8 = [&](int r, float (&v)[8]) {
    const uint4 u = *reinterpret_cast<const uint4*>(tile + ((size_t)r * S + ch0) * 2);
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float2 f = __bfloat1622float2(h[q]);
      v[2 * q] = f.x + addv[2 * q];
      v[2 * q + 1] = f.y + addv[2 * q + 1];
    }
  };
  // per-thread (A, B) partials -> per-group fp64 partial of this CTA, in a
  // fixed order: 32 strided partials per column, a warp shuffle per column,
  // then each group sums its (<= 4) columns
  const int warp = tid >> 5, lane = tid & 31;
  auto fold = [&](double* dst) {
    __syncthreads();
    if (tid < VC * 32) {
      const int jj = tid % VC, q = tid / VC;
      float a = 0.f, b = 0.f;
      for (int k = q; k < rstep; k += 32) {
        const float2 p = part[k * VC + jj];
        a += p.x;
        b += p.y;
      }
      s1[q * VC + jj] = make_float2(a, b);
    }
    __syncthreads();
    if (warp < VC) {
      float2 v = s1[lane * VC + warp];
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        v.x += __shfl_xor_sync(0xffffffffu, v.x, off);
        v.y += __shfl_xor_sync(0xffffffffu, v.y, off);
      }
      if (lane == 0) colsum[warp] = v;
    }
    __syncthreads();
    if (tid < gs) {
      double acc = 0.0;
      for (int jj = 0; jj < VC; ++jj) {
        const int ga = (jj * 8) / cpg;
        const int na = min(8, (ga + 1) * cpg - jj * 8);
        if (ga == tid) acc += colsum[jj].x;
        else if (na < 8 && ga + 1 == tid) acc += colsum[jj].y;
      }
      dst[tid] = acc;
    }
  };
  const double count = (double)hw * cpg;

  // ---- pass 1: sums ---------------------------------------------------------
  {
    float sA = 0.f, sB = 0.f;
    if (active) {
      for (int r = rstart; r < rows; r += rstep) {
        float v[8];
        load8(r, v);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          if (e < nA) sA += v[e];
          else sB += v[e];
        }
      }
    }
    part[tid] = make_float2(sA, sB);
    fold(ex);
  }
  cl_arrive();
  cl_wait();                                          // every CTA's sums visible cluster-wide
  if (tid < gs) {
    double tot = 0.0;
    for (uint32_t r = 0; r < cs; ++r) tot += ld_peer_f64(smem_u32(ex + tid), r);
    stat[tid] = (float)(tot / count);
  }
  __syncthreads();
  // ---- pass 2: centred squares ---------------------------------------------
  const float mA = stat[gA], mB = stat[min(gA + 1, gs - 1)];
  {
    float qA = 0.f, qB = 0.f;
    if (active) {
      for (int r = rstart; r < rows; r += rstep) {
        float v[8];
        load8(r, v);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          if (e < nA) {
            const float d = v[e] - mA;
            qA = fmaf(d, d, qA);
          } else {
            const float d = v[e] - mB;
            qB = fmaf(d, d, qB);
          }
        }
      }
    }
    part[tid] = make_float2(qA, qB);
    fold(ex + kGcMaxGs);
  }
  cl_arrive();
  cl_wait();
  if (tid < gs) {
    double tot = 0.0;
    for (uint32_t r = 0; r < cs; ++r) tot += ld_peer_f64(smem_u32(ex + kGcMaxGs + tid), r);
    stat[kGcMaxGs + tid] = (float)(1.0 / sqrt(tot / count + (double)eps));
  }
  cl_arrive();                                        // this CTA's remote reads are done
  __syncthreads();
  // ---- apply (+ SiLU) in place, then TMA store -------------------------------
  if (active) {
    float a[8], b[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int g = e < nA ? gA : gA + 1;
      const float rs = stat[kGcMaxGs + g], mu = stat[g];
      const int ch = c0 + ch0 + e;
      const float ga = gamma != nullptr ? gamma[ch] : 1.f;
      const float be = beta != nullptr ? beta[ch] : 0.f;
      a[e] = ga * rs;
      b[e] = fmaf(addv[e] - mu, a[e], be);            // y = x*a + (add - mean)*a + beta
      addv[e] = 0.f;
    }
    for (int r = rstart; r < rows; r += rstep) {
      uint4* p = reinterpret_cast<uint4*>(tile + ((size_t)r * S + ch0) * 2);
      uint4 u = *p;
      __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float2 f = __bfloat1622float2(h[q]);
        float y0 = fmaf(f.x, a[2 * q], b[2 * q]);
        float y1 = fmaf(f.y, a[2 * q + 1], b[2 * q + 1]);
        if (SILU) {
          y0 = silu_fast(y0);
          y1 = silu_fast(y1);
        }
        h[q] = __floats2bfloat162_rn(y0, y1);
      }
      *p = u;
    }
  }
  fence_proxy_async();
  __syncthreads();
  if (tid == 0) {
    const uint64_t pol = policy_evict_last();         // the consumer (a conv) reads it next
    for (int k = 0; k < rows; k += br) tma_store_2d(&ymap, c0, row0 + k, smem_u32(tile + (size_t)k * S * 2), pol);
    tma_store_wait_read();
  }
  cl_wait();                                          // peers finished reading this CTA's partials
}

struct GcPlan {
  int S = 0, cs = 0, rows = 0, br = 0;
  size_t smem = 0;
};

bool gc_plan(int64_t n, int64_t hw, int64_t c, int64_t groups, GcPlan& p) {
  const int64_t cpg = c / groups;
  if (cpg < 8) return false;                                   // an 8-channel vector spans <= 2 groups
  if (n * hw * c * 2 > kGcMaxBytes) return false;
  const int64_t S = std::lcm<int64_t>(cpg, 8);                 // whole groups, 16-B rows
  if (S > 256 || c % S != 0 || S / cpg > kGcMaxGs || S / 8 > 32) return false;
  const int64_t rows_max = kGcTileMax / (S * 2);
  const int64_t pairs = n * (c / S);
  int cs = 0;
  for (int d = 1; d <= kGcMaxCs; ++d)
    if (hw % d == 0 && hw / d <= rows_max) {
      cs = d;
      break;
    }
  if (cs == 0) return false;
  // spread over >= ~128 CTAs (one per SM at the big sites) while runs stay >= 64 rows
  while (pairs * cs < kGcTargetCtas && 2 * cs <= kGcMaxCs && hw % (2 * cs) == 0 && hw / (2 * cs) >= 64) cs *= 2;
  const int64_t rows = hw / cs;
  int br = 0;
  for (int d = (int)std::min<int64_t>(256, rows); d >= 1; --d)
    if (rows % d == 0) {
      br = d;
      break;
    }
  if (br < 8 || rows / br > 64) return false;
  if (n * hw > INT32_MAX) return false;
  p.S = (int)S;
  p.cs = cs;
  p.rows = (int)rows;
  p.br = br;
  p.smem = (((size_t)rows * S * 2 + 127) & ~(size_t)127) + kGcExtra;
  return true;
}

template <bool SILU>
int launch_gc(const GcPlan& p, const CUtensorMap& xm, const CUtensorMap& ym, const float* gamma, const float* beta,
              const float* add_nc, int64_t n, int64_t hw, int64_t c, int64_t groups, float eps, cudaStream_t st,
              bool* launched) {
  auto kern = gn_cluster_kernel<SILU>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kGcTileMax + kGcExtra + 256);
    cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)p.cs, (unsigned)(c / p.S), (unsigned)n);
  cfg.blockDim = dim3(kGcThreads, 1, 1);
  cfg.dynamicSmemBytes = p.smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)p.cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int clusters = 0;
  if (cudaOccupancyMaxActiveClusters(&clusters, kern, &cfg) != cudaSuccess || clusters < 1) {
    cudaGetLastError();
    *launched = false;
    return SDB_OK;
  }
  cudaLaunchKernelEx(&cfg, kern, xm, ym, gamma, beta, add_nc, (int)hw, (int)c, (int)(c / groups), p.S, p.rows, p.br,
                     eps);
  *launched = true;
  return check_launch("gn_cluster_kernel");
}

}  // namespace

// Kernel launches a full GroupNorm of this shape costs: 1 (cluster form) or 2.
int gn_launches(int64_t n, int64_t hw, int64_t c, int64_t groups, int dtype) {
  GcPlan p;
  return (g_gn_cluster_mode != 1 && dtype == SDB_BF16 && gc_plan(n, hw, c, groups, p)) ? 1 : 2;
}

// Returns SDB_OK with *launched = true when the single-pass cluster form ran,
// *launched = false when the shape (or the device's cluster occupancy) is not
// eligible — the caller then runs the two-pass form.
int gn_cluster_try(const void* x, void* y, const float* gamma, const float* beta, const float* add_nc, int64_t n,
                   int64_t hw, int64_t c, int64_t groups, float eps, int silu, int dtype, cudaStream_t st,
                   bool* launched) {
  *launched = false;
  if (g_gn_cluster_mode == 1 || dtype != SDB_BF16) return SDB_OK;
  GcPlan p;
  if (!gc_plan(n, hw, c, groups, p)) return SDB_OK;
  EncodeTiledFn enc = encode_fn();
  if (enc == nullptr) return SDB_OK;
  CUtensorMap xm, ym;
  const cuuint64_t dims[2] = {(cuuint64_t)c, (cuuint64_t)(n * hw)};
  const cuuint64_t strides[1] = {(cuuint64_t)(c * 2)};
  const cuuint32_t box[2] = {(cuuint32_t)p.S, (cuuint32_t)p.br};
  const cuuint32_t es[2] = {1, 1};
  if (enc(&xm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(x), dims, strides, box, es,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return SDB_OK;
  if (enc(&ym, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, y, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return SDB_OK;
  if (silu) return launch_gc<true>(p, xm, ym, gamma, beta, add_nc, n, hw, c, groups, eps, st, launched);
  return launch_gc<false>(p, xm, ym, gamma, beta, add_nc, n, hw, c, groups, eps, st, launched);
}

}  // namespace sdb
