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
// i.e. a strided set — but a run of whole pixels is one contiguous span.  So
// each CTA owns a chunk of consecutive pixels of one sample and moves it with
// ONE bulk copy (cp.async.bulk, completion on an mbarrier) into shared memory:
// one memory round trip per CTA instead of a chain of register batches.  The
// SDXL feature maps are 5-63 MB, i.e. a few microseconds of HBM time, so the
// number of dependent round trips per CTA — not bandwidth — was the limit.
//
//   kernel 1  gn_stats_kernel: chunk -> smem; per-thread shifted sums over
//             its 8 channels (shift K = the chunk's first pixel, per group:
//             no cancellation); per-group fold in shared memory; lane 0 turns
//             the chunk's (S1, S2) into raw moments (sum x', sum x'^2) in fp64
//             and adds them with fire-and-forget fp64 atomics.  No counters,
//             no fences, no last-CTA tail, no co-residency requirement (safe
//             next to a concurrent LoRA patch or ControlNet on another stream).
//   kernel 2  gn_apply_kernel: chunk -> smem (L2 hit: kernel 1 read it with
//             an evict-last hint) while the first `groups` threads turn the
//             fp64 moments into mean / rstd (fp64: var = E[x'^2] - mean^2 keeps
//             ~1e-8 relative precision even at |mean| / std = 1e4); then
//             y = act(x * a_c + b_c), a_c = gamma_c*rstd_g,
//             b_c = beta_c + (add_c - mean_g) * a_c, stored straight to HBM.
//
// Accumulator reset without a memset launch: the workspace holds two fp64
// accumulator banks and an epoch word.  Launch L accumulates into bank
// (epoch & 1) and zeroes the other bank (last used by launch L-1, whose apply
// kernel has finished); the apply kernel reads the bank recorded in `cur` and
// its CTA (0, 0) advances the epoch.  Every launch therefore starts on a zero
// bank, including CUDA-graph replays; launches sharing a workspace must be
// ordered on one stream (the C-ABI contract).
//
// Optional add_nc [N][C] (fp32) is added to x before normalisation (x' = x +
// add): the ResNet block's time-embedding projection (h = conv1(x) +
// temb_proj[n, c]) is fused here instead of costing its own read + write of
// the feature map.
#include "common.cuh"
#include "ptx.cuh"

namespace sdb {
namespace {

// 1/d for d in [1, 2^127): bit-trick seed (rel. error <= 5.1%) and two
// Newton steps on the FMA pipe (rel. error <= 6.7e-6, far below bf16's 2^-9)
__device__ __forceinline__ float rcp_nr(float d) {
  float x = __int_as_float(0x7EF311C3 - __float_as_int(d));
  x = x * fmaf(-d, x, 2.f);
  return x * fmaf(-d, x, 2.f);
}

constexpr int kMaxThreads = 512;
constexpr int kMaxN = 16;            // batch (x2 for CFG): serving batch 8 with CFG
constexpr int kMaxGroups = 64;
constexpr int kTileMax = 80 * 1024;          // chunk bytes per CTA (2 CTAs / SM)
// Statistics bank: kSlots independent copies of the (n, group) fp64 moments;
// chunk b of a sample adds into slot b % kSlots, so at most
// ceil(chunks / kSlots) CTAs contend for one L2 atomic address (one copy
// serialised ~150 fp64 atomics per address at the SDXL 128^2 sites).
// The layout is fixed ([kMaxN][slot][kMaxGroups][2]); a launch zeroes the
// idle bank's rows up to the largest batch seen (WsHeader::hwm), so one
// workspace may serve calls of different shapes.
constexpr int kSlots = 8;
constexpr int kBankDoubles = kSlots * kMaxN * kMaxGroups * 2;   // 512 KB
constexpr size_t kWsHeader = 256;            // epoch (u32) | cur (u32) | pad
constexpr size_t kWsBytes = kWsHeader + 2 * (size_t)kBankDoubles * sizeof(double);
__host__ __device__ __forceinline__ size_t bank_index(int slot, int n, int g) {
  return (((size_t)n * kSlots + slot) * kMaxGroups + g) * 2;   // [n][slot][group][2]
}

struct WsHeader {
  unsigned int epoch;
  unsigned int cur;
  unsigned int hwm;   // largest batch ever accumulated: rows >= hwm of both banks are still zero
};

// Zero rows [0, max(hwm, N)) of the idle bank (a grid-strided slice per CTA)
// and publish this launch's bank; returns the bank to accumulate into.
__device__ __forceinline__ double* claim_bank(uint8_t* ws, int nbatch) {
  WsHeader* hdr = reinterpret_cast<WsHeader*>(ws);
  unsigned int epoch, hwmu;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(epoch) : "l"(&hdr->epoch));
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(hwmu) : "l"(&hdr->hwm));
  const int hwm = (int)hwmu;
  const int rows = max(hwm, nbatch);
  double* bank = reinterpret_cast<double*>(ws + kWsHeader) + (size_t)(epoch & 1u) * kBankDoubles;
  double2* o2 = reinterpret_cast<double2*>(reinterpret_cast<double*>(ws + kWsHeader) +
                                           (size_t)((epoch + 1u) & 1u) * kBankDoubles);
  const int cta = blockIdx.y * gridDim.x + blockIdx.x;
  const int ctas = gridDim.x * gridDim.y;
  const int total = rows * kSlots * kMaxGroups;   // double2 entries
  for (int i = cta * blockDim.x + threadIdx.x; i < total; i += ctas * blockDim.x) o2[i] = make_double2(0.0, 0.0);
  if (cta == 0 && threadIdx.x == 0) {
    hdr->cur = epoch & 1u;
    hdr->hwm = (unsigned int)rows;
  }
  return bank;
}

struct GnShape {
  int64_t n, hw, c, groups, cv, cpg, es;
  int rpp, threads;
  int64_t chunks, rows_per_chunk;
  size_t tile_bytes;
};

GnShape gn_shape(int64_t n, int64_t hw, int64_t c, int64_t groups, int64_t es) {
  GnShape s;
  s.n = n; s.hw = hw; s.c = c; s.groups = groups; s.es = es;
  s.cv = c / 8;
  s.cpg = c / groups;
  s.rpp = (int)std::max<int64_t>(1, 256 / s.cv);
  s.threads = (int)(s.cv * s.rpp);
  // ~2 CTAs per SM over the whole batch, each chunk <= kTileMax bytes
  const int64_t want = std::max<int64_t>(1, (2 * kNumSMs + n - 1) / n);
  int64_t rpc = (hw + want - 1) / want;
  rpc = std::min<int64_t>(rpc, std::max<int64_t>(1, kTileMax / (c * es)));
  s.rows_per_chunk = std::max<int64_t>(1, rpc);
  s.chunks = (hw + s.rows_per_chunk - 1) / s.rows_per_chunk;
  s.tile_bytes = (size_t)(s.rows_per_chunk * c * es);
  return s;
}

// Group of each of a thread's 8 channels without a division per channel: one
// 32-bit division for the first, then a running remainder (cpg may be < 8).
__device__ __forceinline__ void channel_groups(int c0, int cpg, int (&g)[8]) {
  int gg = c0 / cpg, rem = c0 - gg * cpg;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    g[j] = gg;
    if (++rem == cpg) { rem = 0; ++gg; }
  }
}

// Thread 0: bulk-copy rows [pbeg, pbeg + m) of one sample into the tile.
template <typename T>
__device__ __forceinline__ void load_chunk(uint8_t* tile, const T* xs, int pbeg, int m, int c, uint64_t* bar,
                                           uint64_t pol) {
  if (threadIdx.x == 0) {
    const uint32_t b = smem_u32(bar);
    mbar_init(b, 1);
    mbar_fence_init();
    const uint32_t bytes = (uint32_t)m * (uint32_t)c * (uint32_t)sizeof(T);
    mbar_expect_tx(b, bytes);
    bulk_g2s(smem_u32(tile), xs + (size_t)pbeg * c, bytes, b, pol);
  }
}

// Apply kernel: the chunk arrives as kSlabs row slabs, each on its own
// mbarrier, so the stores of slab k overlap the arrival of slabs k+1.. (a
// single copy makes every CTA wait for all of its input before its first
// store: read and write phases would never overlap inside the CTA).
constexpr int kSlabs = 4;
template <typename T>
__device__ __forceinline__ void load_chunk_slabs(uint8_t* tile, const T* xs, int pbeg, int m, int c, uint64_t* bars,
                                                 uint64_t pol) {
  if (threadIdx.x == 0) {
    const int rs = (m + kSlabs - 1) / kSlabs;
    for (int k = 0; k < kSlabs; ++k) mbar_init(smem_u32(bars + k), 1);
    mbar_fence_init();
    for (int k = 0; k < kSlabs; ++k) {
      const int r0 = k * rs, r1 = min(m, r0 + rs);
      if (r1 <= r0) {
        mbar_arrive(smem_u32(bars + k));
        continue;
      }
      const uint32_t bytes = (uint32_t)(r1 - r0) * (uint32_t)c * (uint32_t)sizeof(T);
      mbar_expect_tx(smem_u32(bars + k), bytes);
      bulk_g2s(smem_u32(tile + (size_t)r0 * c * sizeof(T)), xs + (size_t)(pbeg + r0) * c, bytes, smem_u32(bars + k),
               pol);
    }
  }
}

// All index math is 32-bit within one sample (host checks hw * c < 2^31).
template <typename T>
__global__ void __launch_bounds__(kMaxThreads)
gn_stats_kernel(const T* __restrict__ x, const float* __restrict__ add_nc, uint8_t* __restrict__ ws, int hw, int c,
                int groups, int cpg, int rows_per_chunk, int rpp, size_t tile_bytes) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar;
  uint8_t* tile = smem;
  float* red1 = reinterpret_cast<float*>(smem + tile_bytes);   // [rpp][c]
  float* red2 = red1 + rpp * c;                                 // [rpp][c]
  const int n = blockIdx.y;
  const int cv = c >> 3;
  const int v = threadIdx.x % cv;
  const int r = threadIdx.x / cv;
  const int c0 = v * 8;
  const T* xs = x + (size_t)n * hw * c;
  const int pbeg = blockIdx.x * rows_per_chunk;
  const int m = min(hw, pbeg + rows_per_chunk) - pbeg;
  // kernel 2 re-reads the chunk right away: keep it in L2
  load_chunk<T>(tile, xs, pbeg, m, c, &bar, policy_evict_last());

  // accumulator bank of this launch; zero the other one (a grid-strided slice per CTA)
  double* bank = claim_bank(ws, gridDim.y);
  double* mine = bank + bank_index(blockIdx.x % kSlots, n, 0);
  int g8[8];
  channel_groups(c0, cpg, g8);
  __syncthreads();            // barrier init visible before anyone waits on it
  mbar_wait(smem_u32(&bar), 0);

  const T* t = reinterpret_cast<const T*>(tile);
  // shift: the chunk's first pixel, first channel of each group
  float2 nK[4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
    nK[i] = make_float2(-to_f32<T>(t[g8[2 * i] * cpg]), -to_f32<T>(t[g8[2 * i + 1] * cpg]));
  float2 s1[4], s2[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) { s1[i] = f2s(0.f); s2[i] = f2s(0.f); }
#pragma unroll 4
  for (int row = r; row < m; row += rpp) {
    const Raw8<T> q = load_raw<T>(t + row * c + c0);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 d = f2add(get_pair<T>(q, i), nK[i]);
      s1[i] = f2add(s1[i], d);
      s2[i] = f2fma(d, d, s2[i]);
    }
  }
  *reinterpret_cast<float4*>(red1 + r * c + c0) = make_float4(s1[0].x, s1[0].y, s1[1].x, s1[1].y);
  *reinterpret_cast<float4*>(red1 + r * c + c0 + 4) = make_float4(s1[2].x, s1[2].y, s1[3].x, s1[3].y);
  *reinterpret_cast<float4*>(red2 + r * c + c0) = make_float4(s2[0].x, s2[0].y, s2[1].x, s2[1].y);
  *reinterpret_cast<float4*>(red2 + r * c + c0 + 4) = make_float4(s2[2].x, s2[2].y, s2[3].x, s2[3].y);
  __syncthreads();
  // fold the rpp pixel rows into row 0 (one thread per channel column)
  if (rpp > 1) {
    for (int ch = threadIdx.x; ch < c; ch += blockDim.x) {
      float a1 = red1[ch], a2 = red2[ch];
      for (int rr = 1; rr < rpp; ++rr) {
        a1 += red1[rr * c + ch];
        a2 += red2[rr * c + ch];
      }
      red1[ch] = a1;
      red2[ch] = a2;
    }
    __syncthreads();
  }
  // one full warp per group: lanes over the group's channels, shuffle-reduce,
  // lane 0 converts the chunk's shifted sums to raw moments of x' = x + add
  // in fp64 (add is per channel, so per channel) and adds them to the bank
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  for (int g = warp; warp < nwarps && g < groups; g += nwarps) {
    const double K = (double)to_f32<T>(t[g * cpg]);
    double m1 = 0.0, m2 = 0.0;
    for (int k = lane; k < cpg; k += 32) {
      const int ch = g * cpg + k;
      const double a = add_nc != nullptr ? (double)add_nc[n * c + ch] : 0.0;
      const double sh = K + a;                       // x' - sh = x - K = d
      const double S1 = (double)red1[ch], S2 = (double)red2[ch];
      m1 += S1 + (double)m * sh;                     // sum x'
      m2 += S2 + sh * (2.0 * S1 + (double)m * sh);   // sum x'^2
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      m1 += __shfl_xor_sync(0xffffffffu, m1, o);
      m2 += __shfl_xor_sync(0xffffffffu, m2, o);
    }
    if (lane == 0) {
      atomicAdd(mine + g * 2 + 0, m1);
      atomicAdd(mine + g * 2 + 1, m2);
    }
  }
}

template <typename T, bool SILU>
__global__ void __launch_bounds__(kMaxThreads)
gn_apply_kernel(const T* x, T* y,  // may alias: every CTA reads its chunk into smem before writing it
                const float* __restrict__ add_nc, uint8_t* __restrict__ ws, const float* __restrict__ gamma,
                const float* __restrict__ beta, int hw, int c, int groups, int cpg, int rows_per_chunk, int rpp,
                float eps) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t bars[kSlabs];
  __shared__ float2 gstat[kMaxGroups];   // (mean, rstd)
  const int n = blockIdx.y;
  const int cv = c >> 3;
  const int v = threadIdx.x % cv;
  const int r = threadIdx.x / cv;
  const int c0 = v * 8;
  const size_t base = (size_t)n * hw * c;
  const int pbeg = blockIdx.x * rows_per_chunk;
  const int m = min(hw, pbeg + rows_per_chunk) - pbeg;
  load_chunk_slabs<T>(smem, x + base, pbeg, m, c, bars, policy_evict_first());

  WsHeader* hdr = reinterpret_cast<WsHeader*>(ws);
  if (threadIdx.x < groups) {
    // one memory round trip: the bank index and every slot of BOTH banks are
    // loaded together (unused slots are zero), then the current bank is summed
    unsigned int cur;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(&hdr->cur));
    const double* banks = reinterpret_cast<const double*>(ws + kWsHeader);
    double2 p0[kSlots], p1[kSlots];
#pragma unroll
    for (int k = 0; k < kSlots; ++k) {
      p0[k] = __ldcg(reinterpret_cast<const double2*>(banks + bank_index(k, n, threadIdx.x)));
      p1[k] = __ldcg(reinterpret_cast<const double2*>(banks + kBankDoubles + bank_index(k, n, threadIdx.x)));
    }
    double m1 = 0.0, m2 = 0.0;
#pragma unroll
    for (int k = 0; k < kSlots; ++k) {
      m1 += (cur & 1u) ? p1[k].x : p0[k].x;
      m2 += (cur & 1u) ? p1[k].y : p0[k].y;
    }
    const double cnt = (double)hw * (double)cpg;
    const double mean = m1 / cnt;
    double var = m2 / cnt - mean * mean;
    if (var < 0.0) var = 0.0;
    gstat[threadIdx.x] = make_float2((float)mean, (float)(1.0 / sqrt(var + (double)eps)));
  }
  // every apply CTA has its bank index already (cur): advancing the epoch
  // here only affects the next launch's stats kernel
  if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) atomicAdd(&hdr->epoch, 1u);
  int g8[8];
  channel_groups(c0, cpg, g8);
  float ga[8], be[8], ad[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    ga[j] = gamma ? gamma[c0 + j] : 1.f;
    be[j] = beta ? beta[c0 + j] : 0.f;
    ad[j] = add_nc ? add_nc[n * c + c0 + j] : 0.f;
  }
  __syncthreads();
  float2 A[4], B[4];
  {
    float a[8], b[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float2 st = gstat[g8[j]];
      a[j] = ga[j] * st.y;
      b[j] = be[j] + (ad[j] - st.x) * a[j];
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      A[i] = make_float2(a[2 * i], a[2 * i + 1]);
      B[i] = make_float2(b[2 * i], b[2 * i + 1]);
    }
  }
  const int slab_rows = (m + kSlabs - 1) / kSlabs;
  int ready = -1;
  const T* t = reinterpret_cast<const T*>(smem);
  T* ys = y + base + (size_t)pbeg * c;
#pragma unroll 4
  for (int row = r; row < m; row += rpp) {
    while (ready < row / slab_rows) mbar_wait(smem_u32(bars + ++ready), 0);
    const Raw8<T> q = load_raw<T>(t + row * c + c0);
    Raw8<T> o;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float2 u = f2fma(get_pair<T>(q, i), A[i], B[i]);
      if (SILU) {   // SiLU(u) = u / (1 + 2^(-u log2 e)) -> 0 as u -> -inf
        // ex2 on the MUFU, the reciprocal on the FMA pipe (rcp_nr): the MUFU
        // was this kernel's busiest pipe with both (ncu: XU 42-62%); 3-5% faster
        // (scripts/gn_cluster_probe.py two-pass column: 24.0 vs 25.0 us at [2,320,128,128])
        float2 w = f2mul(u, f2s(-1.4426950408889634f));
        w.x = fminf(w.x, 126.f);
        w.y = fminf(w.y, 126.f);
        float2 e;
        asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e.x) : "f"(w.x));
        asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e.y) : "f"(w.y));
        e = f2add(e, f2s(1.f));
        if constexpr (sizeof(T) == 4) {   // fp32 output: keep the full-precision MUFU reciprocal
          float2 rc;
          asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rc.x) : "f"(e.x));
          asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rc.y) : "f"(e.y));
          u = f2mul(u, rc);
        } else {                           // 16-bit output: 2 Newton steps (6.7e-6) are far below its ulp
          u = f2mul(u, make_float2(rcp_nr(e.x), rcp_nr(e.y)));
        }
      }
      set_pair<T>(o, i, u);
    }
    store_raw<T>(ys + row * c + c0, o);
  }
}

// ---- K3 + GroupNorm statistics in one pass ---------------------------------
// The input of 29 of SDXL's 46 GN sites is written by K3 (a ResNet / attention
// block's residual add, the up-block concat, a folded conv bias).  This
// kernel IS that K3 pass — out = [hidden (+hb) | skip (+sb) + sum s_i res_i] —
// and accumulates the GroupNorm moments of the rounded output into the GN
// site's workspace bank on the way (fp64 raw moments, same epoch protocol as
// gn_stats_kernel), so that site runs gn_apply_kernel alone: one full read of
// the feature map and one launch less per site.  Per thread the sums are raw
// fp32 over <= ~30 rows (relative error ~1e-6 of sum x^2, i.e. a variance
// error ~1e-6 (1 + mean^2/var) — the UNet's post-residual activations sit at
// |mean| / std = O(1); the two-pass gn_stats_kernel keeps shifted sums for
// arbitrary inputs).  One resident wave of CTAs, each a few row batches whose
// loads are all issued before any store (out may alias skip).
constexpr int kInjMaxRes = 4;
template <typename T>
struct InjArgs {
  const T* res[kInjMaxRes];
  float scale[kInjMaxRes];
};

template <typename T, int NR>
__global__ void __launch_bounds__(kMaxThreads)
inject_gn_kernel(T* out, const T* __restrict__ hidden, const T* skip, InjArgs<T> ra, const float* __restrict__ hb,
                 const float* __restrict__ sb, uint8_t* __restrict__ ws, int hw, int ch, int cs, int groups, int cpg,
                 int rows_per_chunk, int rpp) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int c = ch + cs;
  float* red1 = reinterpret_cast<float*>(smem);   // [rpp][c]
  float* red2 = red1 + rpp * c;                    // [rpp][c]
  const int n = blockIdx.y;
  const int cv = c >> 3, vh = ch >> 3;
  const int v = threadIdx.x % cv;
  const int r = threadIdx.x / cv;
  const int c0 = v * 8;
  const int pbeg = blockIdx.x * rows_per_chunk;
  const int m = min(hw, pbeg + rows_per_chunk) - pbeg;
  const int p0 = n * hw + pbeg;                    // first pixel of the chunk (global pixel index)

  constexpr int kB = 4;
  const bool hid_lane = v < vh;
  const T* src0 = hid_lane ? hidden + c0 : skip + (c0 - ch);
  const int ld0 = hid_lane ? ch : cs;
  const float* bias = hid_lane ? (hb ? hb + c0 : nullptr) : (sb ? sb + (c0 - ch) : nullptr);
  float bv[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) bv[j] = bias ? bias[j] : 0.f;
  float2 s1[4], s2[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) s1[i] = s2[i] = make_float2(0.f, 0.f);
  for (int row0 = r; row0 < m; row0 += kB * rpp) {
    Raw8<T> q0[kB], qr[kB][NR > 0 ? NR : 1];
#pragma unroll
    for (int b = 0; b < kB; ++b) {
      const int row = row0 + b * rpp;
      if (row < m) {
        const size_t p = (size_t)(p0 + row);
        q0[b] = load_raw<T>(src0 + p * ld0);
        if (!hid_lane) {
#pragma unroll
          for (int i = 0; i < NR; ++i) qr[b][i] = load_raw<T>(ra.res[i] + p * cs + (c0 - ch));
        }
      }
    }
#pragma unroll
    for (int b = 0; b < kB; ++b) {
      const int row = row0 + b * rpp;
      if (row < m) {
        float a[8];
        unpack<T>(q0[b], a);
#pragma unroll
        for (int j = 0; j < 8; ++j) a[j] += bv[j];
        if (!hid_lane) {
#pragma unroll
          for (int i = 0; i < NR; ++i) {
            float rb[8];
            unpack<T>(qr[b][i], rb);
#pragma unroll
            for (int j = 0; j < 8; ++j) a[j] = fmaf(ra.scale[i], rb[j], a[j]);
          }
        }
        Raw8<T> q;
        Vec8Half<int>::store(reinterpret_cast<T*>(&q.u), a);   // round once, as stored
        store_raw<T>(out + (size_t)(p0 + row) * c + c0, q);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float2 f = get_pair<T>(q, i);
          s1[i] = f2add(s1[i], f);
          s2[i] = f2fma(f, f, s2[i]);
        }
      }
    }
  }
  *reinterpret_cast<float4*>(red1 + r * c + c0) = make_float4(s1[0].x, s1[0].y, s1[1].x, s1[1].y);
  *reinterpret_cast<float4*>(red1 + r * c + c0 + 4) = make_float4(s1[2].x, s1[2].y, s1[3].x, s1[3].y);
  *reinterpret_cast<float4*>(red2 + r * c + c0) = make_float4(s2[0].x, s2[0].y, s2[1].x, s2[1].y);
  *reinterpret_cast<float4*>(red2 + r * c + c0 + 4) = make_float4(s2[2].x, s2[2].y, s2[3].x, s2[3].y);
  __syncthreads();
  if (rpp > 1) {
    for (int chn = threadIdx.x; chn < c; chn += blockDim.x) {
      float a1 = red1[chn], a2 = red2[chn];
      for (int rr = 1; rr < rpp; ++rr) {
        a1 += red1[rr * c + chn];
        a2 += red2[rr * c + chn];
      }
      red1[chn] = a1;
      red2[chn] = a2;
    }
    __syncthreads();
  }
  // one warp per group: lanes over its channels (fp64), shuffle-reduce, slotted atomics
  double* bank = claim_bank(ws, gridDim.y);
  double* mine = bank + bank_index(blockIdx.x % kSlots, n, 0);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  for (int g = warp; warp < nwarps && g < groups; g += nwarps) {
    double m1 = 0.0, m2 = 0.0;
    for (int k = lane; k < cpg; k += 32) {
      m1 += (double)red1[g * cpg + k];
      m2 += (double)red2[g * cpg + k];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      m1 += __shfl_xor_sync(0xffffffffu, m1, o);
      m2 += __shfl_xor_sync(0xffffffffu, m2, o);
    }
    if (lane == 0) {
      atomicAdd(mine + g * 2 + 0, m1);
      atomicAdd(mine + g * 2 + 1, m2);
    }
  }
}

template <typename T>
void gn_attrs() {
  // opt in to > 48 KB of dynamic shared memory once per device
  static unsigned long long attr_done = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 64 && !((attr_done >> dev) & 1ull)) {
    const int lim = kTileMax + 2 * kMaxThreads * 8 * (int)sizeof(float);
    cudaFuncSetAttribute(gn_stats_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
    cudaFuncSetAttribute(gn_apply_kernel<T, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
    cudaFuncSetAttribute(gn_apply_kernel<T, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
    attr_done |= 1ull << dev;
  }
}

template <typename T>
int run_apply(const T* x, T* y, const float* gamma, const float* beta, const float* add_nc, const GnShape& s,
              float eps, int silu, uint8_t* ws, cudaStream_t st) {
  dim3 grid((unsigned)s.chunks, (unsigned)s.n);
  const int ihw = (int)s.hw, ic = (int)s.c, ig = (int)s.groups, icpg = (int)s.cpg, irows = (int)s.rows_per_chunk;
  if (silu)
    gn_apply_kernel<T, true><<<grid, s.threads, s.tile_bytes, st>>>(x, y, add_nc, ws, gamma, beta, ihw, ic, ig,
                                                                   icpg, irows, s.rpp, eps);
  else
    gn_apply_kernel<T, false><<<grid, s.threads, s.tile_bytes, st>>>(x, y, add_nc, ws, gamma, beta, ihw, ic, ig,
                                                                    icpg, irows, s.rpp, eps);
  return check_launch("gn_apply_kernel");
}

template <typename T>
int run_gn(const void* xv, void* yv, const float* gamma, const float* beta, const float* add_nc, int64_t n,
           int64_t hw, int64_t c, int64_t groups, float eps, int silu, void* wsv, cudaStream_t st, bool stats) {
  const T* x = static_cast<const T*>(xv);
  T* y = static_cast<T*>(yv);
  uint8_t* ws = static_cast<uint8_t*>(wsv);
  GnShape s = gn_shape(n, hw, c, groups, sizeof(T));
  gn_attrs<T>();
  if (stats) {
    dim3 grid((unsigned)s.chunks, (unsigned)n);
    const size_t smem_stats = s.tile_bytes + (size_t)s.rpp * c * 2 * sizeof(float);
    gn_stats_kernel<T><<<grid, s.threads, smem_stats, st>>>(x, add_nc, ws, (int)hw, (int)c, (int)groups, (int)s.cpg,
                                                            (int)s.rows_per_chunk, s.rpp, s.tile_bytes);
    if (int rc = check_launch("gn_stats_kernel")) return rc;
  }
  return run_apply<T>(x, y, gamma, beta, add_nc, s, eps, silu, ws, st);
}

template <typename T>
int run_inject_gn(void* out, const void* hidden, const void* skip, const void* const* res, const float* scales,
                  int n_res, int64_t n, int64_t hw, int64_t ch, int64_t cs, const float* hb, const float* sb,
                  int64_t groups, void* ws, cudaStream_t st) {
  const int64_t c = ch + cs;
  InjArgs<T> ra;
  for (int i = 0; i < kInjMaxRes; ++i) {
    ra.res[i] = i < n_res ? static_cast<const T*>(res[i]) : nullptr;
    ra.scale[i] = i < n_res ? scales[i] : 0.f;
  }
  const int cv = (int)(c / 8);
  const int rpp = std::max(1, 256 / cv);
  const int threads = cv * rpp;
  // one resident wave (~2 CTAs per SM over the batch; measured best against
  // 1, 4, 8 and 16 — the per-CTA statistics epilogue is a serial latency chain)
  const int64_t want = std::max<int64_t>(1, (2 * kNumSMs + n - 1) / n);
  const int64_t rpc = std::max<int64_t>(1, (hw + want - 1) / want);
  const int64_t chunks = (hw + rpc - 1) / rpc;
  const size_t smem = (size_t)2 * rpp * c * sizeof(float);
  dim3 grid((unsigned)chunks, (unsigned)n);
  T* o = static_cast<T*>(out);
  const T* h = static_cast<const T*>(hidden);
  const T* sk = static_cast<const T*>(skip);
  uint8_t* w = static_cast<uint8_t*>(ws);
  const int ihw = (int)hw, ich = (int)ch, ics = (int)cs, ig = (int)groups, icpg = (int)(c / groups), irpc = (int)rpc;
  switch (n_res) {
#define SDB_INJ(NR)                                                                                          \
  case NR:                                                                                                   \
    cudaFuncSetAttribute(inject_gn_kernel<T, NR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);   \
    inject_gn_kernel<T, NR><<<grid, threads, smem, st>>>(o, h, sk, ra, hb, sb, w, ihw, ich, ics, ig, icpg, irpc, \
                                                         rpp);                                               \
    break;
    SDB_INJ(0)
    SDB_INJ(1)
    SDB_INJ(2)
    SDB_INJ(3)
    SDB_INJ(4)
#undef SDB_INJ
    default: return fail(SDB_EINVAL, "residual_inject_gn: at most 4 residuals");
  }
  return check_launch("inject_gn_kernel");
}

}  // namespace

size_t groupnorm_workspace(int64_t n, int64_t hw, int64_t c, int64_t groups) {
  (void)n;
  (void)hw;
  (void)c;
  (void)groups;
  return kWsBytes;
}

static int gn_checks(const void* x, const void* y, int64_t n, int64_t hw, int64_t c, int64_t groups, const void* ws) {
  if (n <= 0 || hw <= 0 || c <= 0 || groups <= 0) return fail(SDB_EINVAL, "groupnorm: empty shape");
  if (n > kMaxN) return fail(SDB_EINVAL, "groupnorm: batch > 16 unsupported");
  if (c % groups != 0) return fail(SDB_EINVAL, "groupnorm: channels not divisible by groups");
  if (groups > kMaxGroups) return fail(SDB_EINVAL, "groupnorm: more than 64 groups");
  if (c % 8 != 0) return fail(SDB_EINVAL, "groupnorm: channels must be a multiple of 8");
  if (c / 8 > kMaxThreads) return fail(SDB_EINVAL, "groupnorm: channels > 4096 unsupported");
  if (n * hw * c >= (int64_t)INT32_MAX - 8 * c)
    return fail(SDB_EINVAL, "groupnorm: the batch must hold < 2^31 elements");
  if (((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y)) & 15) != 0)
    return fail(SDB_EINVAL, "groupnorm: x and y must be 16-byte aligned");
  if (ws == nullptr) return fail(SDB_EINVAL, "groupnorm: workspace is NULL");
  if ((reinterpret_cast<uintptr_t>(ws) & 15) != 0) return fail(SDB_EINVAL, "groupnorm: workspace must be 16-byte aligned");
  return SDB_OK;
}

int gn_cluster_try(const void* x, void* y, const float* gamma, const float* beta, const float* add_nc, int64_t n,
                   int64_t hw, int64_t c, int64_t groups, float eps, int silu, int dtype, cudaStream_t st,
                   bool* launched);

int groupnorm_silu(const void* x, void* y, const float* gamma, const float* beta, const float* add_nc, int64_t n,
                   int64_t hw, int64_t c, int64_t groups, float eps, int silu, int dtype, void* ws,
                   cudaStream_t st, int stats) {
  if (int rc = gn_checks(x, y, n, hw, c, groups, ws)) return rc;
  if (stats) {   // single-pass cluster form where the map fits a cluster's shared memory (gn_cluster.cu)
    bool launched = false;
    if (int rc = gn_cluster_try(x, y, gamma, beta, add_nc, n, hw, c, groups, eps, silu, dtype, st, &launched))
      return rc;
    if (launched) return SDB_OK;
  }
  switch (dtype) {
    case SDB_BF16:
      return run_gn<__nv_bfloat16>(x, y, gamma, beta, add_nc, n, hw, c, groups, eps, silu, ws, st, stats != 0);
    case SDB_F16: return run_gn<__half>(x, y, gamma, beta, add_nc, n, hw, c, groups, eps, silu, ws, st, stats != 0);
    case SDB_F32: return run_gn<float>(x, y, gamma, beta, add_nc, n, hw, c, groups, eps, silu, ws, st, stats != 0);
    default: return fail(SDB_EUNSUP, "groupnorm: unsupported dtype");
  }
}

int residual_inject_gn(void* out, const void* hidden, const void* skip, const void* const* res, const float* scales,
                       int n_res, int64_t n, int64_t hw, int64_t ch, int64_t cs, const float* hidden_bias,
                       const float* skip_bias, int64_t groups, void* ws, int dtype, cudaStream_t st) {
  if (int rc = gn_checks(out, skip, n, hw, ch + cs, groups, ws)) return rc;
  if (n_res < 0 || n_res > kInjMaxRes) return fail(SDB_EINVAL, "residual_inject_gn: n_res must be in [0, 4]");
  if (n_res > 0 && (res == nullptr || scales == nullptr))
    return fail(SDB_EINVAL, "residual_inject_gn: residual pointers / scales missing");
  if (ch % 8 != 0 || cs % 8 != 0 || cs <= 0)
    return fail(SDB_EINVAL, "residual_inject_gn: channel counts must be positive multiples of 8");
  if (ch > 0 && hidden == nullptr) return fail(SDB_EINVAL, "residual_inject_gn: hidden is NULL with ch > 0");
  uintptr_t align = reinterpret_cast<uintptr_t>(hidden) | reinterpret_cast<uintptr_t>(hidden_bias) |
                    reinterpret_cast<uintptr_t>(skip_bias);
  for (int i = 0; i < n_res; ++i) align |= reinterpret_cast<uintptr_t>(res[i]);
  if (align & 15) return fail(SDB_EINVAL, "residual_inject_gn: pointers must be 16-byte aligned");
  switch (dtype) {
    case SDB_BF16:
      return run_inject_gn<__nv_bfloat16>(out, hidden, skip, res, scales, n_res, n, hw, ch, cs, hidden_bias,
                                          skip_bias, groups, ws, st);
    case SDB_F16:
      return run_inject_gn<__half>(out, hidden, skip, res, scales, n_res, n, hw, ch, cs, hidden_bias, skip_bias,
                                   groups, ws, st);
    default: return fail(SDB_EUNSUP, "residual_inject_gn: bf16 / fp16 only");
  }
}

}  // namespace sdb
