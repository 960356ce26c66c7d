// conv_out.cu — K9: the UNet's output convolution (3x3, C -> 4, pad 1) with
// an fp32 result, straight from the bf16 (or fp32) NHWC activations.
//
// Not in the reference (addonsim has no UNet arithmetic); it is
// the last op of every denoising step before K4.  The noise prediction leaves
// the UNet in fp32 because CFG multiplies (eps_c - eps_u) by the guidance
// scale (unet.py decode), and the library route for that — cast the
// [2, 320, 128, 128] activations to fp32, then a TF32 cuDNN convolution with
// 4 output channels — costs ~0.45 ms per SDXL step (a 42 MB fp32 copy plus a
// conv kernel that cannot fill a tensor-core tile with N = 4).
//
// Two forms, both fp32-accumulating:
//  * bf16, C % 32 == 0 (every SD/SDXL UNet): mma.sync m16n8k16 implicit GEMM
//    (conv_out_mma_kernel below; M = 16 pixels, N = 4 real + 4 zero output
//    channels, K = 9C).  SDXL [2, 320, 128, 128]: 21 us vs 68 us for the
//    cast + cuDNN route (scripts/convout_probe.py, CUDA-graph replays, inputs
//    rotated over > L2); max |err| vs an fp64 conv ~5e-6.  The N = 4 GEMM is
//    too narrow for a tcgen05 tile (min N = 8 per CTA with a 128-row M tile
//    would waste the same half, and the op is 0.1% of a step), so the legacy
//    warp-level MMA is the right size here.
//  * everything else (fp32 activations — the fp32 parity configuration — or
//    odd channel counts): fp32 FFMA.  One warp computes a strip of output
//    pixels of one row for all 4 output channels: lanes own channel PAIRS
//    (j = lane, lane + 32, ...), so each load is a coalesced row segment; for
//    each of the 3 input rows the warp loads the strip + 2 halo pixels ONCE
//    and applies the 3 horizontal taps from registers; the per-(tap, pair)
//    weights (8 floats) sit in shared memory.  The STRIP*4 partial sums per
//    lane are reduced across the warp by a halving butterfly that leaves each
//    lane one float2 of the strip's output: a coalesced store.
//
// Roofline: the activation read (N*H*W*C*2 B; 21 MB for SDXL at CFG batch 2,
// just written by K2 so mostly L2-resident); at 21 us the kernel is bound by
// per-warp load -> MMA latency (one strip per warp at this size), not by
// bandwidth.  SDB_K9_VARIANT (probe knob): 1/2 = 128/256-thread MMA CTAs,
// 11/12 = FFMA with 16/8-pixel strips.
#include <type_traits>

#include "common.cuh"

namespace sdb {
namespace {

constexpr int kStrip = 16;        // pixels per warp strip of the widest variant (width granularity)
constexpr int kCout = 4;
constexpr int kWarps = 8;

template <typename T> struct Pair;
template <> struct Pair<__nv_bfloat16> {
  using V = uint32_t;
  __device__ static float2 f2(V v) {
    __nv_bfloat162 b = *reinterpret_cast<__nv_bfloat162*>(&v);
    return __bfloat1622float2(b);
  }
};
template <> struct Pair<float> {
  using V = float2;
  __device__ static float2 f2(V v) { return v; }
};

template <typename T, int STRIP, int MINB>
__global__ void __launch_bounds__(kWarps * 32, MINB)
conv_out_kernel(const T* __restrict__ x, const T* __restrict__ w, const float* __restrict__ bias,
                float* __restrict__ out, int N, int H, int W, int C) {
  pdl_wait();
  constexpr int kStrip = STRIP;
  using P = Pair<T>;
  using V = typename P::V;
  extern __shared__ float4 smem4[];
  float* ws = reinterpret_cast<float*>(smem4);            // [9][C/2][8]
  const int pairs = C >> 1;
  // weight physical layout (Cout, 3, 3, C) (channels_last) -> [tap][pair][(c&1)*4 + o]
  for (int i = threadIdx.x; i < 9 * C * kCout; i += blockDim.x) {   // destination order
    const int k = i & 7;
    const int tp = i >> 3;                     // tap * pairs + pair
    const int tap = tp / pairs;
    const int c = (tp - tap * pairs) * 2 + (k >> 2);
    ws[i] = to_f32<T>(w[((k & 3) * 9 + tap) * C + c]);
  }
  __syncthreads();
  float b[kCout];
#pragma unroll
  for (int o = 0; o < kCout; ++o) b[o] = bias != nullptr ? bias[o] : 0.f;

  const int lane = threadIdx.x & 31;
  const int strips_per_row = W / kStrip;
  const int n_strips = N * H * strips_per_row;
  const V* xv = reinterpret_cast<const V*>(x);
  for (int s = blockIdx.x * kWarps + (threadIdx.x >> 5); s < n_strips; s += gridDim.x * kWarps) {
    const int n = s / (H * strips_per_row);
    const int rem = s - n * H * strips_per_row;
    const int y = rem / strips_per_row;
    const int x0 = (rem - y * strips_per_row) * kStrip;
    float acc[kStrip * kCout];
#pragma unroll
    for (int i = 0; i < kStrip * kCout; ++i) acc[i] = 0.f;
    for (int dy = 0; dy < 3; ++dy) {
      const int yy = y + dy - 1;
      if (yy < 0 || yy >= H) continue;                      // warp-uniform
      const V* row = xv + ((size_t)(n * H + yy) * W) * pairs;
      for (int j = lane; j < pairs; j += 32) {
        V px[kStrip + 2];
#pragma unroll
        for (int p = 0; p < kStrip + 2; ++p) {
          const int xx = x0 + p - 1;
          if (xx >= 0 && xx < W) {
            px[p] = row[(size_t)xx * pairs + j];
          } else {
            px[p] = V{};
          }
        }
#pragma unroll
        for (int dx = 0; dx < 3; ++dx) {
          const float4* wp = reinterpret_cast<const float4*>(ws + ((dy * 3 + dx) * pairs + j) * 8);
          const float4 w0 = wp[0], w1 = wp[1];
#pragma unroll
          for (int p = 0; p < kStrip; ++p) {
            const float2 v = P::f2(px[p + dx]);
            acc[p * 4 + 0] = fmaf(v.x, w0.x, fmaf(v.y, w1.x, acc[p * 4 + 0]));
            acc[p * 4 + 1] = fmaf(v.x, w0.y, fmaf(v.y, w1.y, acc[p * 4 + 1]));
            acc[p * 4 + 2] = fmaf(v.x, w0.z, fmaf(v.y, w1.z, acc[p * 4 + 2]));
            acc[p * 4 + 3] = fmaf(v.x, w0.w, fmaf(v.y, w1.w, acc[p * 4 + 3]));
          }
        }
      }
    }
    // halving butterfly over the STRIP*4 partial sums: each level halves the
    // vector (lanes with bit `off` set keep the upper half); with 64 values
    // lane l ends with values 2l, 2l+1, with 32 values lane pairs (l, l^1)
    // hold the same value l & ~1 ... and one more shuffle level finishes
    constexpr int kVals = kStrip * kCout;
    constexpr int kLevels = kVals == 64 ? 5 : 4;
#pragma unroll
    for (int lvl = 0; lvl < kLevels; ++lvl) {
      const int off = 16 >> lvl;
      const int half = (kVals / 2) >> lvl;
      const bool upper = (lane & off) != 0;
#pragma unroll
      for (int i = 0; i < half; ++i) {
        const float send = upper ? acc[i] : acc[i + half];
        const float keep = upper ? acc[i + half] : acc[i];
        acc[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
      }
    }
    if (kVals == 64) {
      const int p = lane >> 1;
      const int o = (lane & 1) * 2;
      float2 r;
      r.x = acc[0] + b[o];
      r.y = acc[1] + b[o + 1];
      *reinterpret_cast<float2*>(out + ((size_t)(n * H + y) * W + x0 + p) * kCout + o) = r;
    } else {
      // 32 values: after 4 levels lane l holds values 2*(l>>1), +1, partial over lane bit 0
      acc[0] += __shfl_xor_sync(0xffffffffu, acc[0], 1);
      acc[1] += __shfl_xor_sync(0xffffffffu, acc[1], 1);
      if ((lane & 1) == 0) {
        const int v = lane;                    // value index of acc[0]: 2 * (lane >> 1)
        const int p = v >> 2;
        const int o = v & 3;
        float2 r;
        r.x = acc[0] + b[o];
        r.y = acc[1] + b[o + 1];
        *reinterpret_cast<float2*>(out + ((size_t)(n * H + y) * W + x0 + p) * kCout + o) = r;
      }
    }
  }
}

__device__ __forceinline__ void mma_bf16_16816(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                               uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// Tensor-core form (bf16, C % 32 == 0): an implicit GEMM per warp,
// M = 16 output pixels of one row, N = 8 (4 real output channels + 4 zero
// columns), K = 9 taps x C.  The K order inside each 32-channel chunk is
// permuted (identically in A and B — a dot product does not care) so that a
// lane's A registers for two consecutive k16 steps are ONE 16-byte load:
// lane (r = lane/4, q = lane%4) holds channels 32m + 8q .. 8q+7 of pixel r
// (a0|a2 of step 2m, a0|a2 of step 2m+1) and of pixel r+8 (a1|a3): each
// warp load is 8 x 64 contiguous bytes.  The B fragments (the weights,
// 9 x C/16 x 32 lanes x 8 B = 46 KB at C = 320) are built once per CTA in
// shared memory in the same permuted order.  fp32 accumulation: the bf16
// products are exact, so this matches the FFMA form's accuracy class.
template <int THREADS>
__global__ void __launch_bounds__(THREADS, 1)
conv_out_mma_kernel(const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ w,
                    const float* __restrict__ bias, float* __restrict__ out, int N, int H, int W, int C) {
  pdl_wait();
  extern __shared__ uint2 btab[];                 // [9][C/16][32]
  const int KC = C >> 4;
  const int chunks = C >> 5;
  // lanes 16..31 (output columns 4..7) hold zero B fragments
  for (int i = threadIdx.x; i < 9 * KC * 16; i += blockDim.x)
    btab[(i >> 4) * 32 + 16 + (i & 15)] = make_uint2(0u, 0u);
  // one 16-B weight load per (out channel n, tap, 32-channel chunk m, q): channels
  // 32m + 8q .. 8q+7 feed lane 4n+q of k16 steps 2m (first 4) and 2m+1 (last 4):
  // logical k (2q, 2q+1 | 2q+8, 2q+9) of step 2m+h <-> channels 32m + 8q + 4h + (0,1 | 2,3)
  for (int i = threadIdx.x; i < kCout * 9 * chunks * 4; i += blockDim.x) {
    const int q = i & 3;
    const int t = i >> 2;
    const int m = t % chunks;
    const int nt = t / chunks;                    // n * 9 + tap
    const int tap = nt % 9;
    const int n = nt / 9;
    const uint4 v = *reinterpret_cast<const uint4*>(w + (size_t)nt * C + m * 32 + q * 8);
    uint2* d = btab + (size_t)(tap * KC + 2 * m) * 32 + n * 4 + q;
    d[0] = make_uint2(v.x, v.y);
    d[32] = make_uint2(v.z, v.w);
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int r = lane >> 2, q = lane & 3;
  float b0 = 0.f, b1 = 0.f;
  if (bias != nullptr && q < 2) {
    b0 = bias[q * 2];
    b1 = bias[q * 2 + 1];
  }
  const int strips_per_row = W / 16;
  const int n_strips = N * H * strips_per_row;
  const int warps = blockDim.x >> 5;
  for (int s = blockIdx.x * warps + (threadIdx.x >> 5); s < n_strips; s += gridDim.x * warps) {
    const int n = s / (H * strips_per_row);
    const int rem = s - n * H * strips_per_row;
    const int y = rem / strips_per_row;
    const int x0 = (rem - y * strips_per_row) * 16;
    // one accumulator per horizontal tap: three independent MMA chains
    float acc3[3][4] = {};
    for (int dy = 0; dy < 3; ++dy) {
      const int yy = y + dy - 1;
      if (yy < 0 || yy >= H) continue;                        // warp-uniform
      const __nv_bfloat16* rowp = x + (size_t)(n * H + yy) * W * C;
      const uint4* pa[3];
      const uint4* pb[3];
      bool va[3], vb[3];
#pragma unroll
      for (int dx = 0; dx < 3; ++dx) {
        const int xa = x0 + r + dx - 1;
        const int xb = xa + 8;
        va[dx] = xa >= 0;                                      // xa < W always (x0 + 15 + 1 <= W)
        vb[dx] = xb < W;
        pa[dx] = reinterpret_cast<const uint4*>(rowp + (size_t)(va[dx] ? xa : 0) * C + q * 8);
        pb[dx] = reinterpret_cast<const uint4*>(rowp + (size_t)(vb[dx] ? xb : 0) * C + q * 8);
      }
      const uint2* bt = btab + (size_t)(dy * 3 * KC) * 32 + lane;
#pragma unroll 2
      for (int m = 0; m < chunks; ++m) {
#pragma unroll
        for (int dx = 0; dx < 3; ++dx) {
          const uint4 A = va[dx] ? pa[dx][m * 4] : make_uint4(0u, 0u, 0u, 0u);
          const uint4 B = vb[dx] ? pb[dx][m * 4] : make_uint4(0u, 0u, 0u, 0u);
          const uint2 w0 = bt[(dx * KC + 2 * m) * 32];
          const uint2 w1 = bt[(dx * KC + 2 * m + 1) * 32];
          mma_bf16_16816(acc3[dx], A.x, B.x, A.y, B.y, w0.x, w0.y);
          mma_bf16_16816(acc3[dx], A.z, B.z, A.w, B.w, w1.x, w1.y);
        }
      }
    }
    float acc[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[i] = acc3[0][i] + acc3[1][i] + acc3[2][i];
    if (q < 2) {
      float* o = out + ((size_t)(n * H + y) * W + x0 + r) * kCout + q * 2;
      *reinterpret_cast<float2*>(o) = make_float2(acc[0] + b0, acc[1] + b1);
      *reinterpret_cast<float2*>(o + 8 * kCout) = make_float2(acc[2] + b0, acc[3] + b1);
    }
  }
}

template <int THREADS>
int launch_conv_out_mma(const void* x, const void* w, const float* bias, float* out, int N, int H, int W, int C,
                        cudaStream_t st) {
  auto kern = conv_out_mma_kernel<THREADS>;
  constexpr int warps = THREADS / 32;
  const size_t smem = (size_t)9 * (C / 16) * 32 * sizeof(uint2);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  const long strips = (long)N * H * (W / 16);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, warps * 32, smem);
  long grid = (strips + warps - 1) / warps;
  // each CTA builds the 46 KB weight table once: ~16 warps per SM in as few CTAs as possible
  const int want = 512 / THREADS > 0 ? 512 / THREADS : 1;
  const long cap = (long)kNumSMs * (per_sm > 0 ? (per_sm < want ? per_sm : want) : 1);
  if (grid > cap) grid = cap;
  launch_k(kern, (unsigned)grid, warps * 32, smem, st, static_cast<const __nv_bfloat16*>(x),
                                                 static_cast<const __nv_bfloat16*>(w), bias, out, N, H, W, C);
  return check_launch("conv_out_mma_kernel");
}

template <typename T, int STRIP, int MINB>
int launch_conv_out(const void* x, const void* w, const float* bias, float* out, int N, int H, int W, int C,
                    cudaStream_t st) {
  auto kern = conv_out_kernel<T, STRIP, MINB>;
  const size_t smem = (size_t)9 * C * kCout * sizeof(float);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  const long strips = (long)N * H * (W / STRIP);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kWarps * 32, smem);
  long grid = (strips + kWarps - 1) / kWarps;
  const long cap = (long)kNumSMs * (per_sm > 0 ? per_sm : 1);
  if (grid > cap) grid = cap;
  launch_k(kern, (unsigned)grid, kWarps * 32, smem, st, static_cast<const T*>(x), static_cast<const T*>(w), bias, out,
                                                  N, H, W, C);
  return check_launch("conv_out_kernel");
}

int g_conv_variant = -1;

template <typename T>
int run_conv_out(const void* x, const void* w, const float* bias, float* out, int N, int H, int W, int C,
                 cudaStream_t st) {
  if (g_conv_variant < 0) {
    const char* e = getenv("SDB_K9_VARIANT");
    g_conv_variant = e ? atoi(e) : 0;
  }
  if (std::is_same<T, __nv_bfloat16>::value && C % 32 == 0 && g_conv_variant < 10) {
    switch (g_conv_variant) {
      case 1: return launch_conv_out_mma<128>(x, w, bias, out, N, H, W, C, st);
      case 2: return launch_conv_out_mma<256>(x, w, bias, out, N, H, W, C, st);
      default: return launch_conv_out_mma<512>(x, w, bias, out, N, H, W, C, st);
    }
  }
  switch (g_conv_variant - 10) {
    case 1: return launch_conv_out<T, 16, 1>(x, w, bias, out, N, H, W, C, st);
    case 2: return launch_conv_out<T, 8, 2>(x, w, bias, out, N, H, W, C, st);
    default: return launch_conv_out<T, 8, 2>(x, w, bias, out, N, H, W, C, st);
  }
}

}  // namespace

int conv_out(const void* x, const void* w, const float* bias, float* out, int64_t n, int64_t h, int64_t w_,
             int64_t c, int64_t cout, int dtype, cudaStream_t st) {
  if (!x || !w || !out) return fail(SDB_EINVAL, "conv_out: NULL pointer");
  if (cout != kCout) return fail(SDB_EINVAL, "conv_out: only 4 output channels are supported");
  if (n <= 0 || h <= 0 || w_ <= 0 || c <= 0) return fail(SDB_EINVAL, "conv_out: empty shape");
  if (w_ % kStrip != 0) return fail(SDB_EINVAL, "conv_out: width must be a multiple of 16");
  if (c % 2 != 0 || c > 1280) return fail(SDB_EINVAL, "conv_out: channels must be even and <= 1280");
  if (n * h * w_ > (1LL << 30)) return fail(SDB_EINVAL, "conv_out: too many pixels");
  if (dtype == SDB_BF16)
    return run_conv_out<__nv_bfloat16>(x, w, bias, out, (int)n, (int)h, (int)w_, (int)c, st);
  if (dtype == SDB_F32) return run_conv_out<float>(x, w, bias, out, (int)n, (int)h, (int)w_, (int)c, st);
  return fail(SDB_EINVAL, "conv_out: dtype must be bf16 or f32");
}

}  // namespace sdb
