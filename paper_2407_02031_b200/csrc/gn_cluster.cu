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
constexpr int64_t kGcSmallBytes = 6 << 20;     // auto: round 1's form up to here, the streamed form above
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
  pdl_wait();
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
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)p.cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = g_pdl ? 2 : 1;
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


// ---- streamed form (maps up to ~30 MB per wave of clusters) -----------------
// The same one-read / one-write structure, re-organised so the HBM transfers
// overlap the shared-memory passes (round 1's form above loaded the whole
// tile, then ran two passes and a store, each phase waiting on the last):
//
//   * the CTA's tile arrives as `nch` TMA chunks, one mbarrier each; the
//     threads fold chunk k into shifted per-channel fp32 sums (shift = the
//     thread's first value of each channel, no cancellation) while chunks
//     k+1.. are still in flight;
//   * per-thread sums -> fp64 raw moments (+ the per-(n, c) add) -> per-group
//     CTA partials in a fixed order (one warp per group, lanes over the
//     threads of the group's columns, shuffle tree) -> the cluster reads its
//     peers' partials over DSMEM in rank order: deterministic, no atomics,
//     no workspace;
//   * apply + SiLU chunk by chunk in place, each chunk's TMA store issued as
//     soon as it is written, so the store of chunk k overlaps the apply of
//     k+1.
//
// Clusters are independent (one (sample, channel slab) each), so a launch of
// more clusters than fit at once simply runs in waves — nothing waits on a
// co-resident grid.
constexpr int kGsThreads = 1024;
constexpr int kGsMaxChunks = 16;
constexpr int kGsTileMax = 184 * 1024;
constexpr int kGsExtra = kGsThreads * 4 * 8 + 2 * kGcMaxGs * 8 + 2 * kGcMaxGs * 4 + kGsMaxChunks * 8 + 128;

template <bool SILU>
__global__ void __launch_bounds__(kGsThreads, 1)
gn_stream_kernel(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap ymap,
                 const float* __restrict__ gamma, const float* __restrict__ beta, const float* __restrict__ add_nc,
                 int hw, int c, int cpg, int S, int rows, int cr, int nch, float eps) {
  pdl_wait();
  extern __shared__ __align__(128) uint8_t smem[];
  const int tile_bytes = rows * S * 2;
  const int chunk_bytes = cr * S * 2;
  uint8_t* tile = smem;
  double* part = reinterpret_cast<double*>(smem + ((tile_bytes + 127) & ~127));   // [threads][4]
  double* ex = part + kGsThreads * 4;                                             // [2][kGcMaxGs] cluster-visible
  float* stat = reinterpret_cast<float*>(ex + 2 * kGcMaxGs);                     // mean | rstd
  uint64_t* mbar = reinterpret_cast<uint64_t*>(stat + 2 * kGcMaxGs);             // [nch]
  const uint32_t rank = cl_rank(), cs = cl_size();
  const int n = blockIdx.z;
  const int c0 = blockIdx.y * S;
  const int gs = S / cpg;
  const int tid = threadIdx.x;
  const int row0 = n * hw + (int)rank * rows;
  if (tid == 0) {
    prefetch_map(&xmap);
    prefetch_map(&ymap);
    for (int k = 0; k < nch; ++k) mbar_init(smem_u32(mbar + k), 1);
    mbar_fence_init();
  }
  __syncthreads();
  if (tid == 0) {
    const uint64_t pol = policy_evict_first();
    for (int k = 0; k < nch; ++k) {
      const uint32_t bar = smem_u32(mbar + k);
      mbar_expect_tx(bar, (uint32_t)chunk_bytes);
      tma_load_2d(smem_u32(tile + (size_t)k * chunk_bytes), &xmap, c0, row0 + k * cr, bar, pol);
    }
  }
  const int VC = S >> 3;
  const int rstep = kGsThreads / VC;
  const int j = tid % VC;
  const int rstart = tid / VC;
  const bool active = rstart < rstep;
  const int ch0 = j * 8;
  const int gA = ch0 / cpg;
  const int nA = min(8, (gA + 1) * cpg - ch0);        // leading elements in group gA, the rest in gA + 1
  const float* addp = add_nc != nullptr ? add_nc + (size_t)n * c + c0 + ch0 : nullptr;

  // ---- statistics, chunk by chunk as the TMA lands --------------------------
  float K[8], s1[8], s2[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) K[e] = s1[e] = s2[e] = 0.f;
  int mt = 0;
  for (int k = 0; k < nch; ++k) {
    mbar_wait(smem_u32(mbar + k), 0);
    if (!active) continue;
    for (int r = k * cr + rstart; r < (k + 1) * cr; r += rstep) {
      const uint4 u = *reinterpret_cast<const uint4*>(tile + ((size_t)r * S + ch0) * 2);
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
      float v[8];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float2 f = __bfloat1622float2(h[q]);
        v[2 * q] = f.x;
        v[2 * q + 1] = f.y;
      }
      if (mt == 0) {
#pragma unroll
        for (int e = 0; e < 8; ++e) K[e] = v[e];
      }
      ++mt;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float d = v[e] - K[e];
        s1[e] += d;
        s2[e] = fmaf(d, d, s2[e]);
      }
    }
  }
  {  // raw fp64 moments of x' = x + add per channel, collapsed onto the (<= 2) groups of the column
    double pa1 = 0.0, pa2 = 0.0, pb1 = 0.0, pb2 = 0.0;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const double k = K[e], a = s1[e], m = (double)mt, ad = addp != nullptr ? (double)__ldg(addp + e) : 0.0;
      double m1 = a + m * k;
      double m2 = (double)s2[e] + k * (2.0 * a + m * k);
      m2 += ad * (2.0 * m1 + m * ad);
      m1 += m * ad;
      if (e < nA) { pa1 += m1; pa2 += m2; }
      else { pb1 += m1; pb2 += m2; }
    }
    double* pt = part + (size_t)tid * 4;
    pt[0] = active ? pa1 : 0.0;
    pt[1] = active ? pa2 : 0.0;
    pt[2] = active ? pb1 : 0.0;
    pt[3] = active ? pb2 : 0.0;
  }
  __syncthreads();
  const int warp = tid >> 5, lane = tid & 31;
  if (warp < gs) {   // one warp per group: the columns touching it, their threads in a fixed order
    const int g = warp;
    double m1 = 0.0, m2 = 0.0;
    const int jlo = (g * cpg) >> 3, jhi = min(VC - 1, ((g + 1) * cpg - 1) >> 3);
    for (int jj = jlo; jj <= jhi; ++jj) {
      const int ga = (jj * 8) / cpg;
      const int off = ga == g ? 0 : 2;                // this group is the column's A or B part
      for (int q = lane; q < rstep; q += 32) {
        const double* pt = part + (size_t)(jj + q * VC) * 4 + off;
        m1 += pt[0];
        m2 += pt[1];
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      m1 += __shfl_xor_sync(0xffffffffu, m1, o);
      m2 += __shfl_xor_sync(0xffffffffu, m2, o);
    }
    if (lane == 0) {
      ex[g] = m1;
      ex[kGcMaxGs + g] = m2;
    }
  }
  cl_arrive();
  cl_wait();                                          // every CTA's partials visible cluster-wide
  if (tid < gs) {
    double t1 = 0.0, t2 = 0.0;
    for (uint32_t r = 0; r < cs; ++r) {
      t1 += ld_peer_f64(smem_u32(ex + tid), r);
      t2 += ld_peer_f64(smem_u32(ex + kGcMaxGs + tid), r);
    }
    const double count = (double)hw * cpg;
    const double mean = t1 / count;
    double var = t2 / count - mean * mean;
    var = var < 0.0 ? 0.0 : var;
    stat[tid] = (float)mean;
    stat[kGcMaxGs + tid] = (float)(1.0 / sqrt(var + (double)eps));
  }
  cl_arrive();                                        // this CTA's remote reads are done
  __syncthreads();
  // ---- apply (+ SiLU) in place, chunk by chunk, each chunk stored at once ---
  float a[8], b[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const int g = e < nA ? gA : min(gA + 1, gs - 1);
    const float rs = stat[kGcMaxGs + g], mu = stat[g];
    const int ch = c0 + ch0 + e;
    const float ga = gamma != nullptr ? __ldg(gamma + ch) : 1.f;
    const float be = beta != nullptr ? __ldg(beta + ch) : 0.f;
    a[e] = ga * rs;
    const float ad = addp != nullptr ? __ldg(addp + e) : 0.f;
    b[e] = fmaf(ad - mu, a[e], be);                   // y = x*a + (add - mean)*a + beta
  }
  const uint64_t spol = policy_evict_last();          // the consumer (a conv) reads it next
  for (int k = 0; k < nch; ++k) {
    if (active) {
      for (int r = k * cr + rstart; r < (k + 1) * cr; r += rstep) {
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
    if (tid == 0) tma_store_2d(&ymap, c0, row0 + k * cr, smem_u32(tile + (size_t)k * chunk_bytes), spol);
  }
  if (tid == 0) tma_store_wait_read();
  cl_wait();                                          // peers finished reading this CTA's partials
}

struct GsPlan {
  int S = 0, cs = 0, rows = 0, cr = 0, nch = 0;
  int clusters = 0, active = 0;
  size_t smem = 0;
};

int g_gs_force_S = 0, g_gs_force_cs = 0;   // sweep overrides (SDB_GN_SLAB="S,cs"), 0 = planner

template <bool SILU>
int gs_active_clusters(int cs, size_t smem) {
  static int cache[17][16] = {};
  const int sb = (int)std::min<size_t>(15, smem / (16 * 1024));
  if (cache[cs][sb] != 0) return cache[cs][sb] > 0 ? cache[cs][sb] : 0;
  auto kern = gn_stream_kernel<SILU>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kGsTileMax + kGsExtra + 256);
    cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)cs, 1, 1);
  cfg.blockDim = dim3(kGsThreads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int clusters = 0;
  if (cudaOccupancyMaxActiveClusters(&clusters, kern, &cfg) != cudaSuccess) {
    cudaGetLastError();
    clusters = 0;
  }
  cache[cs][sb] = clusters > 0 ? clusters : -1;
  return clusters;
}

bool gs_plan(int64_t n, int64_t hw, int64_t c, int64_t groups, bool silu, GsPlan& best) {
  const int64_t cpg = c / groups;
  if (cpg < 8 || n * hw > INT32_MAX) return false;           // an 8-channel vector spans <= 2 groups
  const int64_t base = std::lcm<int64_t>(cpg, 8);             // whole groups, 16-B rows
  double best_cost = 0.0;
  bool found = false;
  for (int64_t S = base; S <= 256 && S <= c; S += base) {
    if (c % S != 0 || S / cpg > kGcMaxGs) continue;
    if (g_gs_force_S != 0 && S != g_gs_force_S) continue;
    for (int cs = 1; cs <= kGcMaxCs; cs *= 2) {
      if (g_gs_force_cs != 0 && cs != g_gs_force_cs) continue;
      if (hw % cs != 0) continue;
      const int64_t rows = hw / cs;
      const int64_t tile = rows * S * 2;
      if (tile > kGsTileMax) continue;
      int nch = 0;
      for (int d = 4; d <= kGsMaxChunks; ++d)
        if (rows % d == 0 && rows / d <= 256) {
          nch = d;
          break;
        }
      if (nch == 0) continue;
      const size_t smem = (((size_t)tile + 127) & ~(size_t)127) + kGsExtra;
      const int act = silu ? gs_active_clusters<true>(cs, smem) : gs_active_clusters<false>(cs, smem);
      if (act < 1) continue;
      const int64_t clusters = n * (c / S);
      const int64_t waves = (clusters + act - 1) / act;
      // critical path ~ waves x the per-CTA tile (each SM streams its tile in
      // and out); ties -> wider slabs (longer DRAM rows), then smaller clusters
      const double cost = (double)waves * (double)tile * (1.0 + 0.02 * (256.0 / (double)S)) * (1.0 + 0.01 * cs);
      if (!found || cost < best_cost) {
        found = true;
        best_cost = cost;
        best.S = (int)S;
        best.cs = cs;
        best.rows = (int)rows;
        best.nch = nch;
        best.cr = (int)(rows / nch);
        best.clusters = (int)clusters;
        best.active = act;
        best.smem = smem;
      }
    }
  }
  return found;
}

template <bool SILU>
int launch_gs(const GsPlan& p, const CUtensorMap& xm, const CUtensorMap& ym, const float* gamma, const float* beta,
              const float* add_nc, int64_t n, int64_t hw, int64_t c, int64_t groups, float eps, cudaStream_t st) {
  auto kern = gn_stream_kernel<SILU>;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)p.cs, (unsigned)(c / p.S), (unsigned)n);
  cfg.blockDim = dim3(kGsThreads, 1, 1);
  cfg.dynamicSmemBytes = p.smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)p.cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = g_pdl ? 2 : 1;
  cudaLaunchKernelEx(&cfg, kern, xm, ym, gamma, beta, add_nc, (int)hw, (int)c, (int)(c / groups), p.S, p.rows, p.cr,
                     p.nch, eps);
  return check_launch("gn_stream_kernel");
}

}  // namespace

// Which form a full GroupNorm of this shape takes: 1 = round 1's cluster
// form (maps <= 6 MB), 2 = the streamed cluster form, 0 = the two-pass form.
// Modes: 0 auto, 1 force two-pass, 2 only the round-1 cluster form, 3 only the
// streamed form (tests / probes).
static int gn_form(int64_t n, int64_t hw, int64_t c, int64_t groups, int dtype, int silu, GcPlan* gc, GsPlan* gs) {
  if (g_gn_cluster_mode == 1 || dtype != SDB_BF16) return 0;
  static bool env = false;
  if (!env) {
    env = true;
    if (const char* e = getenv("SDB_GN_SLAB")) sscanf(e, "%d,%d", &g_gs_force_S, &g_gs_force_cs);
  }
  GcPlan p1;
  GsPlan p2;
  const bool v1 = g_gn_cluster_mode != 3 && gc_plan(n, hw, c, groups, p1);
  if (v1 && g_gn_cluster_mode == 2) {
    if (gc) *gc = p1;
    return 1;
  }
  if (g_gn_cluster_mode == 2) return 0;
  if (v1 && g_gn_cluster_mode == 0 && n * hw * c * 2 <= kGcSmallBytes) {
    if (gc) *gc = p1;
    return 1;
  }
  // auto: the streamed form only where its clusters run in one wave (measured,
  // scripts/gn_stream_probe.py: [2,640,64,64] 14.6 us vs 23.4 two-pass; with
  // two or more waves each wave's load -> exchange -> store chain serialises:
  // [2,320,128,128] 16 clusters of 8 vs 15 co-resident, 37 us vs 27 two-pass)
  if (gs_plan(n, hw, c, groups, silu != 0, p2) && (g_gn_cluster_mode == 3 || p2.clusters <= p2.active)) {
    if (gs) *gs = p2;
    return 2;
  }
  if (v1) {
    if (gc) *gc = p1;
    return 1;
  }
  return 0;
}

// Kernel launches a full GroupNorm of this shape costs: 1 (a cluster form) or 2.
bool gn_resident_auto(int64_t n, int64_t hw, int64_t c, int64_t groups, int silu, int dtype);

int gn_launches(int64_t n, int64_t hw, int64_t c, int64_t groups, int dtype) {
  if (gn_resident_auto(n, hw, c, groups, 1, dtype)) return 1;
  return gn_form(n, hw, c, groups, dtype, 1, nullptr, nullptr) != 0 ? 1 : 2;
}

// Returns SDB_OK with *launched = true when a single-pass cluster form ran,
// *launched = false when the shape (or the device's cluster occupancy) is not
// eligible — the caller then runs the two-pass form.
int gn_cluster_try(const void* x, void* y, const float* gamma, const float* beta, const float* add_nc, int64_t n,
                   int64_t hw, int64_t c, int64_t groups, float eps, int silu, int dtype, cudaStream_t st,
                   bool* launched) {
  *launched = false;
  GcPlan p1;
  GsPlan p2;
  const int form = gn_form(n, hw, c, groups, dtype, silu, &p1, &p2);
  if (form == 0) return SDB_OK;
  EncodeTiledFn enc = encode_fn();
  if (enc == nullptr) return SDB_OK;
  CUtensorMap xm, ym;
  const cuuint64_t dims[2] = {(cuuint64_t)c, (cuuint64_t)(n * hw)};
  const cuuint64_t strides[1] = {(cuuint64_t)(c * 2)};
  const cuuint32_t box[2] = {(cuuint32_t)(form == 1 ? p1.S : p2.S), (cuuint32_t)(form == 1 ? p1.br : p2.cr)};
  const cuuint32_t es[2] = {1, 1};
  if (enc(&xm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(x), dims, strides, box, es,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return SDB_OK;
  if (enc(&ym, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, y, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return SDB_OK;
  if (form == 2) {
    *launched = true;
    if (silu) return launch_gs<true>(p2, xm, ym, gamma, beta, add_nc, n, hw, c, groups, eps, st);
    return launch_gs<false>(p2, xm, ym, gamma, beta, add_nc, n, hw, c, groups, eps, st);
  }
  if (silu) return launch_gc<true>(p1, xm, ym, gamma, beta, add_nc, n, hw, c, groups, eps, st, launched);
  return launch_gc<false>(p1, xm, ym, gamma, beta, add_nc, n, hw, c, groups, eps, st, launched);
}

// The streamed form's plan for a shape (probes / tests): S, cs, rows, chunk
// rows, chunks, clusters, co-resident clusters; returns 0 when not eligible.
int gn_stream_plan(int64_t n, int64_t hw, int64_t c, int64_t groups, int* out7) {
  GsPlan p;
  if (!gs_plan(n, hw, c, groups, true, p)) return 0;
  const int v[7] = {p.S, p.cs, p.rows, p.cr, p.nch, p.clusters, p.active};
  for (int i = 0; i < 7; ++i) out7[i] = v[i];
  return 1;
}

}  // namespace sdb
