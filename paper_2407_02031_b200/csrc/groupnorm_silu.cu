// groupnorm_silu.cu — K2: GroupNorm (+ SiLU) over NHWC feature maps.
//
// The reference has no arithmetic for this op: it is only the 1.072
// sub-multiplier of addonsim/model.py:66-70 (the paper's fused GN+SiLU,
// PAPER.md:572-576, "35 such combinations" in SDXL).  Semantics follow
// torch.nn.GroupNorm followed by SiLU: per (sample, group) mean and biased
// variance over (C/G channels x H x W), eps inside the rsqrt, per-channel
// affine, then y * sigmoid(y).
//
// Layout: NHWC (torch channels_last) because the convolutions around every
// GN site run channels_last on cuDNN; a group is C/G channels of every pixel,
// i.e. a strided set.  Thread mapping keeps the 16-byte vector lanes fixed on
// channels: blockDim = CV * rpp with CV = C/8 vector columns and rpp pixel
// rows per pass, so each thread always owns the same 8 channels and
// accumulates them in registers — fully coalesced 16 B loads, no atomics on
// the data path.  Every thread handles exactly kRowsPerThread pixel rows per
// chunk and issues all of their loads before consuming any (the kernel is a
// streaming pass: memory-level parallelism is the whole game).
//
//   kernel 1  gn_stats_kernel: per (n, chunk) shifted sums S1 = sum(x'-K_g),
//             S2 = sum((x'-K_g)^2) reduced per group in shared memory and
//             added to per-(n, g) fp64 accumulators; the LAST CTA of each
//             sample (threadfence + counter) turns them into mean / rstd and
//             re-zeroes them — no separate finalize launch, no serial tail,
//             no co-residency requirement (safe next to a concurrent LoRA
//             patch or ControlNet on another stream).
//   kernel 2  gn_apply_kernel: y = act(x * a_c + b_c), a_c = gamma_c*rstd_g,
//             b_c = beta_c + (add_c - mean_g) * a_c.
// Kernel 2 re-reads x right after kernel 1 streamed it; at SDXL sizes the
// tensor (<= 63 MB at CFG batch 2) stays in the 126 MB L2, so HBM traffic
// stays close to the algorithmic one read + one write.
//
// Optional add_nc [N][C] (fp32) is added to x before normalisation (x' = x +
// add): the ResNet block's time-embedding projection (h = conv1(x) +
// temb_proj[n, c]) is fused here instead of costing its own read + write of
// the feature map.  The shift K_g = x[n, pixel 0, g*cpg] is one constant per
// group, so the variance is shift-invariant and free of cancellation.
#include "common.cuh"

namespace sdb {
namespace {

constexpr int kMaxThreads = 512;
constexpr int kMaxGroups = 64;
constexpr int kRowsPerThread = 8;

// 8 consecutive elements of T held as raw registers until they are consumed
template <typename T> struct Raw8 { uint4 u; };
template <> struct Raw8<float> { float4 a, b; };

template <typename T>
__device__ __forceinline__ Raw8<T> load_raw(const T* p) {
  Raw8<T> r;
  r.u = *reinterpret_cast<const uint4*>(p);
  return r;
}
template <>
__device__ __forceinline__ Raw8<float> load_raw<float>(const float* p) {
  Raw8<float> r;
  r.a = *reinterpret_cast<const float4*>(p);
  r.b = *reinterpret_cast<const float4*>(p + 4);
  return r;
}
template <typename T>
__device__ __forceinline__ void unpack(const Raw8<T>& r, float (&v)[8]) {
  const T* h = reinterpret_cast<const T*>(&r.u);
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = to_f32<T>(h[i]);
}
template <>
__device__ __forceinline__ void unpack<float>(const Raw8<float>& r, float (&v)[8]) {
  v[0] = r.a.x; v[1] = r.a.y; v[2] = r.a.z; v[3] = r.a.w;
  v[4] = r.b.x; v[5] = r.b.y; v[6] = r.b.z; v[7] = r.b.w;
}

struct GnShape {
  int64_t n, hw, c, groups, cv, cpg;
  int rpp, threads;
  int64_t chunks, rows_per_chunk;
};

GnShape gn_shape(int64_t n, int64_t hw, int64_t c, int64_t groups) {
  GnShape s;
  s.n = n; s.hw = hw; s.c = c; s.groups = groups;
  s.cv = c / 8;
  s.cpg = c / groups;
  s.rpp = (int)std::max<int64_t>(1, 256 / s.cv);
  s.threads = (int)(s.cv * s.rpp);
  // ~2 CTAs per SM over the whole batch; each thread walks its chunk in
  // batches of kRowsPerThread rows (all loads of a batch in flight), so the
  // per-CTA fixed costs (shift, reduction, accumulator atomics) amortise
  const int64_t batch = (int64_t)s.rpp * kRowsPerThread;
  const int64_t want = std::max<int64_t>(1, (2 * kNumSMs + n - 1) / n);
  s.chunks = std::max<int64_t>(1, std::min<int64_t>(want, (hw + batch - 1) / batch));
  s.rows_per_chunk = (hw + s.chunks - 1) / s.chunks;
  s.chunks = (hw + s.rows_per_chunk - 1) / s.rows_per_chunk;
  return s;
}

// workspace: counters[n] (uint) | acc[n][group][2] (double) — both zero at rest —
// | stats[n][group][2] (float)
template <typename T>
__global__ void __launch_bounds__(kMaxThreads)
gn_stats_kernel(const T* __restrict__ x, const float* __restrict__ add_nc, double* __restrict__ acc,
                float* __restrict__ stats, unsigned int* __restrict__ counters, int64_t hw, int64_t c,
                int64_t groups, int64_t cpg, int64_t rows_per_chunk, int64_t chunks, int rpp, float eps) {
  extern __shared__ float red[];  // [rpp][c][2]
  __shared__ bool is_last;
  const int64_t n = blockIdx.y;
  const int64_t chunk = blockIdx.x;
  const int cv = (int)(c / 8);
  const int v = threadIdx.x % cv;
  const int r = threadIdx.x / cv;
  const int64_t c0 = (int64_t)v * 8;
  const T* xs = x + n * hw * c;
  const int64_t p0 = chunk * rows_per_chunk + r;
  const int64_t p1 = min(hw, chunk * rows_per_chunk + rows_per_chunk);

  // d = x' - K_g = x - (K_g - add_c)
  float K[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    K[j] = to_f32<T>(xs[((c0 + j) / cpg) * cpg]);
    if (add_nc != nullptr) K[j] -= add_nc[n * c + c0 + j];
  }
  float s1[8], s2[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) { s1[j] = 0.f; s2[j] = 0.f; }
  for (int64_t pb = p0; pb < p1; pb += (int64_t)rpp * kRowsPerThread) {
    // every load of the batch first
    Raw8<T> buf[kRowsPerThread];
#pragma unroll
    for (int u = 0; u < kRowsPerThread; ++u) {
      const int64_t p = pb + (int64_t)u * rpp;
      if (p < p1) buf[u] = load_raw<T>(xs + p * c + c0);
    }
#pragma unroll
    for (int u = 0; u < kRowsPerThread; ++u) {
      if (pb + (int64_t)u * rpp < p1) {
        float a[8];
        unpack<T>(buf[u], a);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float d = a[j] - K[j];
          s1[j] += d;
          s2[j] = fmaf(d, d, s2[j]);
        }
      }
    }
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    red[((int64_t)r * c + c0 + j) * 2 + 0] = s1[j];
    red[((int64_t)r * c + c0 + j) * 2 + 1] = s2[j];
  }
  __syncthreads();
  // per-group partials of this chunk go straight into fp64 accumulators: the
  // partials are fp32 sums of similar magnitude, so their fp64 sum is exact in
  // practice and the mean / rstd rounded to fp32 do not depend on arrival order
  // one warp per group: lanes sum the group's (rpp x cpg) partials, shuffle-reduce
  {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    const int per_group = rpp * (int)cpg;
    if (warp < nwarps) {
      for (int64_t g = warp; g < groups; g += nwarps) {
        float t1 = 0.f, t2 = 0.f;
        for (int e = lane; e < per_group; e += 32) {
          const int rr = e / (int)cpg;
          const int64_t ch = g * cpg + e % (int)cpg;
          t1 += red[((int64_t)rr * c + ch) * 2 + 0];
          t2 += red[((int64_t)rr * c + ch) * 2 + 1];
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          t1 += __shfl_xor_sync(0xffffffffu, t1, o);
          t2 += __shfl_xor_sync(0xffffffffu, t2, o);
        }
        if (lane == 0) {
          atomicAdd(acc + (n * groups + g) * 2 + 0, (double)t1);
          atomicAdd(acc + (n * groups + g) * 2 + 1, (double)t2);
        }
      }
    }
  }
  // ---- the last CTA of this sample finalises (no extra launch) ----
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int done = atomicAdd(counters + n, 1u);
    is_last = (done == (unsigned int)chunks - 1);
  }
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  for (int64_t g = threadIdx.x; g < groups; g += blockDim.x) {
    double* a = acc + (n * groups + g) * 2;
    const double t1 = __ldcg(a), t2 = __ldcg(a + 1);
    const double cnt = (double)hw * (double)cpg;
    const double Kg = (double)to_f32<T>(xs[g * cpg]);
    const double dm = t1 / cnt;
    double var = t2 / cnt - dm * dm;
    if (var < 0.0) var = 0.0;
    stats[(n * groups + g) * 2 + 0] = (float)(Kg + dm);
    stats[(n * groups + g) * 2 + 1] = (float)(1.0 / sqrt(var + (double)eps));
    a[0] = 0.0;   // accumulators and counter are back at zero for the next launch / graph replay
    a[1] = 0.0;
  }
  if (threadIdx.x == 0) counters[n] = 0u;
}

template <typename T, bool SILU>
__global__ void __launch_bounds__(kMaxThreads)
gn_apply_kernel(const T* x, T* y,  // may alias: same-thread read-then-write
                const float* __restrict__ add_nc, const float* __restrict__ stats,
                const float* __restrict__ gamma, const float* __restrict__ beta, int64_t hw, int64_t c,
                int64_t groups, int64_t cpg, int64_t rows_per_chunk, int rpp) {
  const int64_t n = blockIdx.y;
  const int64_t chunk = blockIdx.x;
  const int cv = (int)(c / 8);
  const int v = threadIdx.x % cv;
  const int r = threadIdx.x / cv;
  const int64_t c0 = (int64_t)v * 8;
  const T* xs = x + n * hw * c;
  T* ys = y + n * hw * c;
  const int64_t p0 = chunk * rows_per_chunk + r;
  const int64_t p1 = min(hw, chunk * rows_per_chunk + rows_per_chunk);
  float A[8], B[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int64_t ch = c0 + j;
    const int64_t g = ch / cpg;
    const float mean = stats[(n * groups + g) * 2 + 0];
    const float rstd = stats[(n * groups + g) * 2 + 1];
    const float ga = gamma ? gamma[ch] : 1.f;
    const float be = beta ? beta[ch] : 0.f;
    const float ad = add_nc ? add_nc[n * c + ch] : 0.f;
    A[j] = ga * rstd;
    B[j] = be + (ad - mean) * A[j];
  }
  for (int64_t pb = p0; pb < p1; pb += (int64_t)rpp * kRowsPerThread) {
    Raw8<T> buf[kRowsPerThread];
#pragma unroll
    for (int u = 0; u < kRowsPerThread; ++u) {
      const int64_t p = pb + (int64_t)u * rpp;
      if (p < p1) buf[u] = load_raw<T>(xs + p * c + c0);
    }
#pragma unroll
    for (int u = 0; u < kRowsPerThread; ++u) {
      const int64_t p = pb + (int64_t)u * rpp;
      if (p < p1) {
        float a[8];
        unpack<T>(buf[u], a);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          float t = fmaf(a[j], A[j], B[j]);
          if (SILU) t = __fdividef(t, 1.f + __expf(-t));   // -> 0 as t -> -inf
          a[j] = t;
        }
        Vec8<T>::store(ys + p * c + c0, a);
      }
    }
  }
}

template <typename T>
int run_gn(const void* xv, void* yv, const float* gamma, const float* beta, const float* add_nc, int64_t n,
           int64_t hw, int64_t c, int64_t groups, float eps, int silu, void* ws, cudaStream_t st) {
  const T* x = static_cast<const T*>(xv);
  T* y = static_cast<T*>(yv);
  GnShape s = gn_shape(n, hw, c, groups);
  unsigned int* counters = static_cast<unsigned int*>(ws);
  double* acc = reinterpret_cast<double*>(static_cast<uint8_t*>(ws) + 256);
  float* stats = reinterpret_cast<float*>(acc + n * groups * 2);
  dim3 grid((unsigned)s.chunks, (unsigned)n);
  size_t smem = (size_t)s.rpp * c * 2 * sizeof(float);
  if (smem > 48 * 1024) {
    cudaFuncSetAttribute(gn_stats_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  }
  gn_stats_kernel<T><<<grid, s.threads, smem, st>>>(x, add_nc, acc, stats, counters, hw, c, groups, s.cpg,
                                                    s.rows_per_chunk, s.chunks, s.rpp, eps);
  if (int rc = check_launch("gn_stats_kernel")) return rc;
  if (silu)
    gn_apply_kernel<T, true><<<grid, s.threads, 0, st>>>(x, y, add_nc, stats, gamma, beta, hw, c, groups, s.cpg,
                                                         s.rows_per_chunk, s.rpp);
  else
    gn_apply_kernel<T, false><<<grid, s.threads, 0, st>>>(x, y, add_nc, stats, gamma, beta, hw, c, groups, s.cpg,
                                                          s.rows_per_chunk, s.rpp);
  return check_launch("gn_apply_kernel");
}

}  // namespace

size_t groupnorm_workspace(int64_t n, int64_t hw, int64_t c, int64_t groups) {
  (void)hw;
  (void)c;
  return 256 + (size_t)(n * groups * 2) * (sizeof(double) + sizeof(float));
}

int groupnorm_silu(const void* x, void* y, const float* gamma, const float* beta, const float* add_nc, int64_t n,
                   int64_t hw, int64_t c, int64_t groups, float eps, int silu, int dtype, void* ws,
                   cudaStream_t st) {
  if (n <= 0 || hw <= 0 || c <= 0 || groups <= 0) return fail(SDB_EINVAL, "groupnorm: empty shape");
  if (n > 64) return fail(SDB_EINVAL, "groupnorm: batch > 64 unsupported");
  if (c % groups != 0) return fail(SDB_EINVAL, "groupnorm: channels not divisible by groups");
  if (groups > kMaxGroups) return fail(SDB_EINVAL, "groupnorm: more than 64 groups");
  if (c % 8 != 0) return fail(SDB_EINVAL, "groupnorm: channels must be a multiple of 8");
  if (c / 8 > kMaxThreads) return fail(SDB_EINVAL, "groupnorm: channels > 4096 unsupported");
  if (((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y)) & 15) != 0)
    return fail(SDB_EINVAL, "groupnorm: x and y must be 16-byte aligned");
  if (ws == nullptr) return fail(SDB_EINVAL, "groupnorm: workspace is NULL");
  switch (dtype) {
    case SDB_BF16: return run_gn<__nv_bfloat16>(x, y, gamma, beta, add_nc, n, hw, c, groups, eps, silu, ws, st);
    case SDB_F16: return run_gn<__half>(x, y, gamma, beta, add_nc, n, hw, c, groups, eps, silu, ws, st);
    case SDB_F32: return run_gn<float>(x, y, gamma, beta, add_nc, n, hw, c, groups, eps, silu, ws, st);
    default: return fail(SDB_EUNSUP, "groupnorm: unsupported dtype");
  }
}

}  // namespace sdb
