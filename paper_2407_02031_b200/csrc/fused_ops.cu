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
#include "common.cuh"

namespace sdb {
namespace {

// Each thread owns kGegluVec 8-element vectors spaced one grid apart and issues
// all of their loads (value and gate halves) before computing any.
constexpr int kGegluVec = 4;

// 2-d mapping, no integer division: blockIdx.x picks a 8*blockDim-wide column
// slice of the row, each thread walks rows grid-stride (kGegluVec rows per
// round, all loads issued first).
template <typename T>
__global__ void __launch_bounds__(128)
geglu_kernel(const T* __restrict__ proj, T* __restrict__ out, int64_t rows, int64_t f) {
  const int64_t c = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 8;
  if (c >= f) return;
  const int64_t rstride = gridDim.y;
  for (int64_t m0 = blockIdx.y; m0 < rows; m0 += rstride * kGegluVec) {
    float h[kGegluVec][8], g[kGegluVec][8];
#pragma unroll
    for (int u = 0; u < kGegluVec; ++u) {
      const int64_t m = m0 + u * rstride;
      if (m < rows) {
        Vec8<T>::load(proj + m * 2 * f + c, h[u]);
        Vec8<T>::load(proj + m * 2 * f + f + c, g[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < kGegluVec; ++u) {
      const int64_t m = m0 + u * rstride;
      if (m < rows) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
          h[u][j] = h[u][j] * (0.5f * g[u][j] * (1.f + erff(g[u][j] * 0.70710678118654752f)));
        Vec8<T>::store(out + m * f + c, h[u]);
      }
    }
  }
}

// NV = vectors of 8 per lane (C = 256 * NV max per warp pass)
template <typename T>
__device__ __forceinline__ void unpack8(const uint4& u, float (&v)[8]) {
  if constexpr (sizeof(T) == 2) {
    const T* h = reinterpret_cast<const T*>(&u);
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = to_f32<T>(h[i]);
  }
}

// 16-bit T: every load of the row (x, d, gamma, beta) is issued before any is
// consumed — one memory round trip per row instead of three dependent ones.
template <typename T, int NV>
__global__ void __launch_bounds__(128)
add_layernorm_kernel(T* x, const T* __restrict__ d, T* __restrict__ y, const T* __restrict__ gamma,
                     const T* __restrict__ beta, int64_t rows, int64_t c, float eps) {
  const int lane = threadIdx.x & 31;
  constexpr bool kHalf = sizeof(T) == 2;
  // gamma / beta are the same for every row: loaded once per warp
  uint4 gq[NV], bq[NV];
  if constexpr (kHalf) {
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      const int64_t col = (int64_t)(k * 32 + lane) * 8;
      if (col < c) {
        gq[k] = __ldg(reinterpret_cast<const uint4*>(gamma + col));
        bq[k] = __ldg(reinterpret_cast<const uint4*>(beta + col));
      }
    }
  }
  const int64_t warps_total = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); row < rows;
       row += warps_total) {
  T* xr = x + row * c;
  float v[NV][8];
  float sum = 0.f;
  uint4 xq[NV], dq[NV];
  if constexpr (kHalf) {
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      const int64_t col = (int64_t)(k * 32 + lane) * 8;
      if (col < c) {
        xq[k] = *reinterpret_cast<const uint4*>(xr + col);
        if (d != nullptr) dq[k] = *reinterpret_cast<const uint4*>(d + row * c + col);
      }
    }
  }
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const int64_t col = (int64_t)(k * 32 + lane) * 8;
    if (col < c) {
      if constexpr (kHalf) unpack8<T>(xq[k], v[k]); else Vec8<T>::load(xr + col, v[k]);
      if (d != nullptr) {
        float dv[8];
        if constexpr (kHalf) unpack8<T>(dq[k], dv); else Vec8<T>::load(d + row * c + col, dv);
#pragma unroll
        for (int j = 0; j < 8; ++j) v[k][j] += dv[j];
        // the residual stream is stored in T: round once, normalise the stored value
#pragma unroll
        for (int j = 0; j < 8; ++j) v[k][j] = to_f32<T>(from_f32<T>(v[k][j]));
        Vec8<T>::store(xr + col, v[k]);
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) sum += v[k][j];
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  const float mean = sum / (float)c;
  float sq = 0.f;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const int64_t col = (int64_t)(k * 32 + lane) * 8;
    if (col < c) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float t = v[k][j] - mean;
        sq = fmaf(t, t, sq);
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
  const float rstd = rsqrtf(sq / (float)c + eps);
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const int64_t col = (int64_t)(k * 32 + lane) * 8;
    if (col < c) {
      float ga[8], be[8], o[8];
      if constexpr (kHalf) {
        unpack8<T>(gq[k], ga);
        unpack8<T>(bq[k], be);
      } else {
        Vec8<T>::load(gamma + col, ga);
        Vec8<T>::load(beta + col, be);
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) o[j] = fmaf((v[k][j] - mean) * rstd, ga[j], be[j]);
      Vec8<T>::store(y + row * c + col, o);
    }
  }
  }  // rows of this warp
}

template <typename T>
int run_geglu(const void* proj, void* out, int64_t rows, int64_t f, cudaStream_t st) {
  const unsigned gx = (unsigned)((f / 8 + 127) / 128);
  // ~16 CTAs of 128 threads per SM in flight overall
  const int64_t want_y = std::max<int64_t>(1, (int64_t)kNumSMs * 16 / gx);
  const unsigned gy = (unsigned)std::min<int64_t>(std::min<int64_t>(want_y, (rows + kGegluVec - 1) / kGegluVec), 65535);
  geglu_kernel<T><<<dim3(gx, std::max(gy, 1u)), 128, 0, st>>>(static_cast<const T*>(proj), static_cast<T*>(out),
                                                               rows, f);
  return check_launch("geglu_kernel");
}

template <typename T>
int run_add_ln(void* x, const void* d, void* y, const void* gamma, const void* beta, int64_t rows, int64_t c,
               float eps, cudaStream_t st) {
  // 4 warps per 128-thread CTA, each warp walks rows grid-stride (gamma / beta
  // loaded once); ~8 CTAs per SM
  const unsigned grid = (unsigned)std::min<int64_t>((rows + 3) / 4, (int64_t)kNumSMs * 8);
  T* xp = static_cast<T*>(x);
  const T* dp = static_cast<const T*>(d);
  T* yp = static_cast<T*>(y);
  const T* gp = static_cast<const T*>(gamma);
  const T* bp = static_cast<const T*>(beta);
  const int nv = (int)((c / 8 + 31) / 32);
  switch (nv) {
    case 1: add_layernorm_kernel<T, 1><<<grid, 128, 0, st>>>(xp, dp, yp, gp, bp, rows, c, eps); break;
    case 2: add_layernorm_kernel<T, 2><<<grid, 128, 0, st>>>(xp, dp, yp, gp, bp, rows, c, eps); break;
    case 3: add_layernorm_kernel<T, 3><<<grid, 128, 0, st>>>(xp, dp, yp, gp, bp, rows, c, eps); break;
    case 4: add_layernorm_kernel<T, 4><<<grid, 128, 0, st>>>(xp, dp, yp, gp, bp, rows, c, eps); break;
    case 5: add_layernorm_kernel<T, 5><<<grid, 128, 0, st>>>(xp, dp, yp, gp, bp, rows, c, eps); break;
    case 6: add_layernorm_kernel<T, 6><<<grid, 128, 0, st>>>(xp, dp, yp, gp, bp, rows, c, eps); break;
    case 7: add_layernorm_kernel<T, 7><<<grid, 128, 0, st>>>(xp, dp, yp, gp, bp, rows, c, eps); break;
    case 8: add_layernorm_kernel<T, 8><<<grid, 128, 0, st>>>(xp, dp, yp, gp, bp, rows, c, eps); break;
    case 9: add_layernorm_kernel<T, 9><<<grid, 128, 0, st>>>(xp, dp, yp, gp, bp, rows, c, eps); break;
    case 10: add_layernorm_kernel<T, 10><<<grid, 128, 0, st>>>(xp, dp, yp, gp, bp, rows, c, eps); break;
    default: return fail(SDB_EINVAL, "add_layernorm: channels must be <= 2560");
  }
  return check_launch("add_layernorm_kernel");
}

}  // namespace

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

}  // namespace sdb
