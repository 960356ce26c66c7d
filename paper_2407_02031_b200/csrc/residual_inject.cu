// residual_inject.cu — K3: ControlNet residual injection fused with the
// up-block skip concat (NHWC).
//
//   out[p, 0:ch]     = hidden[p, :] (+ hidden_bias[:])
//   out[p, ch:ch+cs] = skip[p, :] (+ skip_bias[:]) + sum_i s_i * res_i[p, :]
//
// The optional fp32 per-channel biases fold the bias of the convolution that
// produced hidden / skip (cuDNN's channels_last bf16 convolutions would add it
// in a separate broadcast pass), so a conv -> K3 pair costs no extra pass.
//
// The paper adds every ControlNet's down/mid outputs to the UNet's skip
// connections and middle block; the reference
// simulator models that sum as free and charges only the
// transfer (addonsim/model.py:151-158).  In an NHWC UNet the skip is consumed
// by torch.cat([hidden, skip], dim=C), itself a full read+write of both
// tensors, so the injection is folded into that copy: one read of hidden,
// skip and each residual, one write of the concat buffer — the algorithmic
// minimum.  With ch == 0 / hidden == NULL it is the in-place mid-block add.
// out may alias skip (in-place mid add): each element is read and written
// by the same thread, so no __restrict__ on those two.
// Sums are in fp32 in the order skip, res_0, res_1, ... (deterministic).
#include "common.cuh"

namespace sdb {
namespace {

constexpr int kMaxRes = 8;

template <typename T>
struct ResArgs {
  const T* res[kMaxRes];
  float scale[kMaxRes];
};

__device__ __forceinline__ void add_bias8(float (&a)[8], const float* __restrict__ b) {
  const float4 b0 = __ldg(reinterpret_cast<const float4*>(b));
  const float4 b1 = __ldg(reinterpret_cast<const float4*>(b) + 1);
  a[0] += b0.x; a[1] += b0.y; a[2] += b0.z; a[3] += b0.w;
  a[4] += b1.x; a[5] += b1.y; a[6] += b1.z; a[7] += b1.w;
}

// 32-bit index math (callers guarantee pixels * (ch + cs) / 8 < 2^31): the
// emulated 64-bit division per vector cost more than the memory traffic.
template <typename T, int NR>
__global__ void __launch_bounds__(256)
residual_inject_kernel(T* out, const T* __restrict__ hidden,
                       const T* skip, ResArgs<T> ra, int n_res,
                       int64_t pixels, int64_t ch, int64_t cs,
                       const float* __restrict__ hbias, const float* __restrict__ sbias) {
  pdl_wait();
  const uint32_t vh = (uint32_t)(ch / 8), vs = (uint32_t)(cs / 8), vrow = vh + vs;
  const uint32_t total = (uint32_t)(pixels * vrow);
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int64_t p = i / vrow;
    const int64_t v = i % vrow;
    float a[8];
    if (v < vh) {
      Vec8<T>::load(hidden + p * ch + v * 8, a);
      if (hbias) add_bias8(a, hbias + v * 8);
    } else {
      const int64_t off = p * cs + (v - vh) * 8;
      Vec8<T>::load(skip + off, a);
      if (sbias) add_bias8(a, sbias + (v - vh) * 8);
      const int nr = NR > 0 ? NR : n_res;
#pragma unroll
      for (int r = 0; r < (NR > 0 ? NR : kMaxRes); ++r) {
        if (r < nr) {
          float b[8];
          Vec8<T>::load(ra.res[r] + off, b);
#pragma unroll
          for (int j = 0; j < 8; ++j) a[j] = fmaf(ra.scale[r], b[j], a[j]);
        }
      }
    }
    Vec8<T>::store(out + p * (ch + cs) + v * 8, a);
  }
}

template <typename T>
int run_inject(void* out, const void* hidden, const void* skip, const void* const* res,
               const float* scales, int n_res, int64_t pixels, int64_t ch, int64_t cs,
               const float* hb, const float* sb, cudaStream_t st) {
  ResArgs<T> ra;
  for (int i = 0; i < kMaxRes; ++i) {
    ra.res[i] = i < n_res ? static_cast<const T*>(res[i]) : nullptr;
    ra.scale[i] = i < n_res ? scales[i] : 0.f;
  }
  const int64_t total = pixels * ((ch + cs) / 8);
  if (total + (int64_t)kNumSMs * 8 * 256 >= (int64_t)INT32_MAX)
    return fail(SDB_EINVAL, "residual_inject: tensor too large (>= 2^31 vectors)");
  int64_t grid = (total + 255) / 256;
  const int64_t cap = (int64_t)kNumSMs * 8;
  if (grid > cap) grid = cap;
  if (grid < 1) grid = 1;
  T* o = static_cast<T*>(out);
  const T* h = static_cast<const T*>(hidden);
  const T* s = static_cast<const T*>(skip);
  switch (n_res) {
    case 0: launch_k(residual_inject_kernel<T, 0>, (unsigned)grid, 256, 0, st, o, h, s, ra, 0, pixels, ch, cs, hb, sb); break;
    case 1: launch_k(residual_inject_kernel<T, 1>, (unsigned)grid, 256, 0, st, o, h, s, ra, 1, pixels, ch, cs, hb, sb); break;
    case 2: launch_k(residual_inject_kernel<T, 2>, (unsigned)grid, 256, 0, st, o, h, s, ra, 2, pixels, ch, cs, hb, sb); break;
    case 3: launch_k(residual_inject_kernel<T, 3>, (unsigned)grid, 256, 0, st, o, h, s, ra, 3, pixels, ch, cs, hb, sb); break;
    default: launch_k(residual_inject_kernel<T, -1>, (unsigned)grid, 256, 0, st, o, h, s, ra, n_res, pixels, ch, cs, hb, sb); break;
  }
  return check_launch("residual_inject_kernel");
}

}  // namespace

int residual_inject(void* out, const void* hidden, const void* skip, const void* const* res,
                    const float* scales, int n_res, int64_t pixels, int64_t ch, int64_t cs,
                    const float* hidden_bias, const float* skip_bias, int dtype, cudaStream_t st) {
  if (n_res < 0 || n_res > kMaxRes) return fail(SDB_EINVAL, "residual_inject: n_res must be in [0, 8]");
  if (n_res > 0 && (res == nullptr || scales == nullptr))
    return fail(SDB_EINVAL, "residual_inject: residual pointers / scales missing");
  if (ch % 8 != 0 || cs % 8 != 0 || cs <= 0)
    return fail(SDB_EINVAL, "residual_inject: channel counts must be positive multiples of 8");
  if (ch > 0 && hidden == nullptr) return fail(SDB_EINVAL, "residual_inject: hidden is NULL with ch > 0");
  uintptr_t align = reinterpret_cast<uintptr_t>(out) | reinterpret_cast<uintptr_t>(skip) |
                    reinterpret_cast<uintptr_t>(hidden);
  for (int i = 0; i < n_res; ++i) align |= reinterpret_cast<uintptr_t>(res[i]);
  if (align & 15) return fail(SDB_EINVAL, "residual_inject: pointers must be 16-byte aligned");
  if ((reinterpret_cast<uintptr_t>(hidden_bias) | reinterpret_cast<uintptr_t>(skip_bias)) & 15)
    return fail(SDB_EINVAL, "residual_inject: bias vectors must be 16-byte aligned fp32");
  if (hidden_bias && ch == 0) return fail(SDB_EINVAL, "residual_inject: hidden_bias without hidden channels");
  if (pixels == 0) return SDB_OK;
  switch (dtype) {
    case SDB_BF16: return run_inject<__nv_bfloat16>(out, hidden, skip, res, scales, n_res, pixels, ch, cs, hidden_bias, skip_bias, st);
    case SDB_F16: return run_inject<__half>(out, hidden, skip, res, scales, n_res, pixels, ch, cs, hidden_bias, skip_bias, st);
    case SDB_F32: return run_inject<float>(out, hidden, skip, res, scales, n_res, pixels, ch, cs, hidden_bias, skip_bias, st);
    default: return fail(SDB_EUNSUP, "residual_inject: unsupported dtype");
  }
}

}  // namespace sdb
