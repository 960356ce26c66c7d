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
// accumulates them in registers — fully coalesced 16 B loads, no atomics.
//
//   pass 1  gn_partial_kernel : shifted sums  S1 = sum(x-K_g), S2 = sum((x-K_g)^2)
//                                per (n, chunk, channel-vector) -> reduced per group
//   pass 2  gn_finalize_kernel: fp64 combine over chunks -> mean, rstd per (n, g)
//   pass 3  gn_apply_kernel   : y = act(x * a_c + b_c), a_c = gamma_c*rstd_g,
//                                b_c = beta_c - mean_g*a_c
// Pass 3 re-reads x right after pass 1 touched it; at SDXL sizes the tensor
// (<= 63 MB at CFG batch 2) stays in the 126 MB L2, so HBM traffic stays close
// to the algorithmic one read + one write.  The shift K_g (the group's first
// element) keeps the one-pass variance free of cancellation.
//
// Optional add_nc [N][C] (fp32) is added to x before normalisation: the
// ResNet block's time-embedding projection (h = conv1(x) + temb_proj[n, c])
// is fused here instead of costing its own read + write of the feature map.
#include "common.cuh"

namespace sdb {
namespace {

constexpr int kMaxThreads = 512;

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
  s.rpp = (int)std::max<int64_t>(1, 384 / s.cv);
  s.threads = (int)(s.cv * s.rpp);
  // ~4 waves of CTAs over 148 SMs across the whole batch
  int64_t target = (4 * kNumSMs + n - 1) / n;
  int64_t max_chunks = (hw + s.rpp - 1) / s.rpp;
  s.chunks = std::max<int64_t>(1, std::min<int64_t>(target, max_chunks));
  s.rows_per_chunk = (hw + s.chunks - 1) / s.chunks;
  s.chunks = (hw + s.rows_per_chunk - 1) / s.rows_per_chunk;
  return s;
}

// partial[n][chunk][group][2]
template <typename T>
__global__ void gn_partial_kernel(const T* __restrict__ x, const float* __restrict__ add_nc,
                                  float* __restrict__ partial,
                                  int64_t hw, int64_t c, int64_t groups, int64_t cpg,
                                  int64_t rows_per_chunk, int64_t chunks, int rpp) {
  extern __shared__ float red[];  // [rpp][c][2] then reused
  const int64_t n = blockIdx.y;
  const int64_t chunk = blockIdx.x;
  const int cv = (int)(c / 8);
  const int v = threadIdx.x % cv;
  const int r = threadIdx.x / cv;
  const int64_t c0 = (int64_t)v * 8;
  const T* xs = x + n * hw * c;

  // per-channel shift = first element of its group (pixel 0, channel g*cpg)
  // (the optional per-(n,c) input bias is folded into the shift: d = x - (K - a))
  float K[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    K[j] = to_f32<T>(xs[((c0 + j) / cpg) * cpg]);
    if (add_nc != nullptr) K[j] -= add_nc[n * c + c0 + j];
  }

  float s1[8], s2[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) { s1[j] = 0.f; s2[j] = 0.f; }

  const int64_t p0 = chunk * rows_per_chunk;
  const int64_t p1 = min(hw, p0 + rows_per_chunk);
  int64_t p = p0 + r;
  // 2-deep unroll for memory-level parallelism
  for (; p + rpp < p1; p += 2 * rpp) {
    float a[8], b[8];
    Vec8<T>::load(xs + p * c + c0, a);
    Vec8<T>::load(xs + (p + rpp) * c + c0, b);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float d = a[j] - K[j];
      s1[j] += d; s2[j] = fmaf(d, d, s2[j]);
      float e = b[j] - K[j];
      s1[j] += e; s2[j] = fmaf(e, e, s2[j]);
    }
  }
  for (; p < p1; p += rpp) {
    float a[8];
    Vec8<T>::load(xs + p * c + c0, a);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float d = a[j] - K[j];
      s1[j] += d; s2[j] = fmaf(d, d, s2[j]);
    }
  }
  // reduce over the rpp row lanes: red[r][ch][2]
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    red[((int64_t)r * c + c0 + j) * 2 + 0] = s1[j];
    red[((int64_t)r * c + c0 + j) * 2 + 1] = s2[j];
  }
  __syncthreads();
  // one thread per group sums its cpg channels over rpp rows
  for (int64_t g = threadIdx.x; g < groups; g += blockDim.x) {
    float t1 = 0.f, t2 = 0.f;
    for (int rr = 0; rr < rpp; ++rr)
      for (int64_t ch = g * cpg; ch < (g + 1) * cpg; ++ch) {
        t1 += red[((int64_t)rr * c + ch) * 2 + 0];
        t2 += red[((int64_t)rr * c + ch) * 2 + 1];
      }
    float* out = partial + ((n * chunks + chunk) * groups + g) * 2;
    out[0] = t1;
    out[1] = t2;
  }
}

// stats[n][g] = {mean, rstd}
template <typename T>
__global__ void gn_finalize_kernel(const T* __restrict__ x, const float* __restrict__ partial,
                                   float* __restrict__ stats, int64_t n_total, int64_t hw,
                                   int64_t c, int64_t groups, int64_t cpg, int64_t chunks,
                                   float eps) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n_total * groups) return;
  const int64_t n = idx / groups, g = idx % groups;
  double t1 = 0.0, t2 = 0.0;
  for (int64_t ch = 0; ch < chunks; ++ch) {
    const float* pp = partial + ((n * chunks + ch) * groups + g) * 2;
    t1 += pp[0];
    t2 += pp[1];
  }
  const double cnt = (double)hw * (double)cpg;
  const double K = to_f32<T>(x[n * hw * c + g * cpg]);
  const double dm = t1 / cnt;
  double var = t2 / cnt - dm * dm;
  if (var < 0.0) var = 0.0;
  stats[idx * 2 + 0] = (float)(K + dm);
  stats[idx * 2 + 1] = (float)(1.0 / sqrt(var + (double)eps));
}

template <typename T, bool SILU>
__global__ void gn_apply_kernel(const T* x, T* y,  // may alias: same-thread read-then-write
                                const float* __restrict__ add_nc,
                                const float* __restrict__ stats, const float* __restrict__ gamma,
                                const float* __restrict__ beta, int64_t hw, int64_t c,
                                int64_t groups, int64_t cpg, int64_t rows_per_chunk, int rpp) {
  const int64_t n = blockIdx.y;
  const int64_t chunk = blockIdx.x;
  const int cv = (int)(c / 8);
  const int v = threadIdx.x % cv;
  const int r = threadIdx.x / cv;
  const int64_t c0 = (int64_t)v * 8;
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
  const T* xs = x + n * hw * c;
  T* ys = y + n * hw * c;
  const int64_t p0 = chunk * rows_per_chunk;
  const int64_t p1 = min(hw, p0 + rows_per_chunk);
  for (int64_t p = p0 + r; p < p1; p += rpp) {
    float a[8];
    Vec8<T>::load(xs + p * c + c0, a);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float t = fmaf(a[j], A[j], B[j]);
      if (SILU) t = t / (1.f + expf(-t));
      a[j] = t;
    }
    Vec8<T>::store(ys + p * c + c0, a);
  }
}

template <typename T>
int run_gn(const void* xv, void* yv, const float* gamma, const float* beta, const float* add_nc, int64_t n,
           int64_t hw, int64_t c, int64_t groups, float eps, int silu, void* ws,
           cudaStream_t st) {
  const T* x = static_cast<const T*>(xv);
  T* y = static_cast<T*>(yv);
  GnShape s = gn_shape(n, hw, c, groups);
  float* partial = static_cast<float*>(ws);
  float* stats = partial + n * s.chunks * groups * 2;
  dim3 grid((unsigned)s.chunks, (unsigned)n);
  size_t smem = (size_t)s.rpp * c * 2 * sizeof(float);
  if (smem > 48 * 1024) {
    cudaFuncSetAttribute(gn_partial_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  }
  gn_partial_kernel<T><<<grid, s.threads, smem, st>>>(x, add_nc, partial, hw, c, groups, s.cpg,
                                                      s.rows_per_chunk, s.chunks, s.rpp);
  if (int rc = check_launch("gn_partial_kernel")) return rc;
  int64_t ng = n * groups;
  gn_finalize_kernel<T><<<(unsigned)((ng + 127) / 128), 128, 0, st>>>(x, partial, stats, n, hw, c, groups,
                                                                    s.cpg, s.chunks, eps);
  if (int rc = check_launch("gn_finalize_kernel")) return rc;
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
  GnShape s = gn_shape(n, hw, c, groups);
  return (size_t)(n * s.chunks * groups * 2 + n * groups * 2) * sizeof(float);
}

int groupnorm_silu(const void* x, void* y, const float* gamma, const float* beta,
                   const float* add_nc, int64_t n,
                   int64_t hw, int64_t c, int64_t groups, float eps, int silu, int dtype,
                   void* ws, cudaStream_t st) {
  if (n <= 0 || hw <= 0 || c <= 0 || groups <= 0) return fail(SDB_EINVAL, "groupnorm: empty shape");
  if (c % groups != 0) return fail(SDB_EINVAL, "groupnorm: channels not divisible by groups");
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
