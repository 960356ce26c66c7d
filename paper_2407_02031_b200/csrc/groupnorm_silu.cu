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
// a strided set, so every CTA owns a run of whole pixels of one sample (one
// contiguous span) and every thread a fixed 8-channel (16 B) lane of it.
//
//   kernel 1  gn_stats_kernel: ~2 CTAs of <= 512 threads per SM over the
//             batch; a CTA is rpp pixel rows x (C/8) lanes, and CTA b of a
//             sample takes row blocks b, b + S, b + 2S, ... (interleaved: at
//             any moment the grid sweeps one contiguous stretch of the map,
//             measured ~15% faster than a contiguous span per CTA,
//             scripts/micro/stream_micro.cu); each thread keeps kStatsUnroll
//             16-B loads in flight and accumulates shifted sums (shift = the
//             CTA's first pixel per group: no cancellation); rows folded in
//             shared memory, one warp per group turns the CTA's sums into
//             fp64 raw moments of x' = x + add and adds them to the site's
//             bank as exact fixed-point integers (red.global.add of an int64
//             integer part + an int64 2^-40 fraction): integer addition is
//             associative, so the statistics are bit-for-bit the same
//             whatever order the CTAs land in (round 1 added fp64 with
//             atomics: order-dependent), and no CTA waits for a reduction.
//   kernel 2  gn_apply_kernel: per CTA a table a_c = gamma_c rstd_g,
//             b_c = beta_c + (add_c - mean_g) a_c for its sample in shared
//             memory, then y = act(x a_c + b_c) streamed (same interleaved
//             row blocks, ~4 CTAs per SM) with kApplyUnroll vectors in flight
//             per thread; the map is an L2 hit after kernel 1.
//
// Workspace (per call site, zeroed once, 256 KB, any shape): a header (epoch,
// current bank, high-water batch, arrival counter) and two banks of
// [16 samples][64 groups] fixed-point (sum x', sum x'^2).  Producer launches
// alternate banks (see producer_bank); K3's fused form (inject_gn_kernel)
// is a producer too, so its consumer GN site runs kernel 2 alone.

// Optional add_nc [N][C] (fp32) is added to x before normalisation (x' = x +
// add): the ResNet block's time-embedding projection (h = conv1(x) +
// temb_proj[n, c]) is fused here instead of costing its own read + write of
// the feature map.
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "ptx.cuh"

namespace sdb {
namespace {

constexpr int kMaxThreads = 512;
constexpr int kMaxN = 16;            // batch (x2 for CFG): serving batch 8 with CFG
constexpr int kMaxGroups = 64;
constexpr int kStatsUnroll = 4;      // 16-B loads in flight per thread (stats; 8 measured slower, scripts/micro/gnstats_micro.cu)
constexpr int kApplyUnroll = 4;      // vectors in flight per thread (apply)
// Workspace: header | 2 banks of [kMaxN][kMaxGroups] x {sum x, sum x^2}, each
// an exact fixed-point pair (int64 integer part, int64 2^-40 fraction).
constexpr size_t kWsHeader = 256;
// Each of a group's 4 words (sum hi, sum lo, sum-of-squares hi, lo) in its
// own 32-B sector: the L2 serialises atomics per sector, and every producer
// CTA adds to the same group words (scripts/k3_probe.py: with the words
// packed in one sector the tail grew to ~16 us at 1184 CTAs).
constexpr int kWordPad = 4;                       // longs between a group's words
constexpr int kGroupStride = 4 * kWordPad;        // longs per (sample, group)
constexpr int kBankWords = kMaxN * kMaxGroups * kGroupStride;
constexpr size_t kWsBytes = kWsHeader + 2 * (size_t)kBankWords * sizeof(long long);
constexpr double kFracScale = 1099511627776.0;        // 2^40
constexpr size_t kRsCntOffset = 128;   // the resident form's per-sample arrival counts: header bytes [128, 256) = [2 banks][16 samples] u32
struct WsHeader {
  unsigned int epoch;      // bank of the next producer launch = epoch & 1
  unsigned int cur;        // bank the last producer launch filled (what apply reads)
  unsigned int hwm;        // rows (samples) any launch ever used: rows >= hwm of both banks are zero
  unsigned int arrivals;   // CTAs of the running producer launch that finished
};

// Decomposition of one (n, hw, c) map for a kernel with ~ctas_per_sm CTAs of
// <= max_threads threads per SM: a CTA is rpp pixel rows x cv lanes; a
// sample's rows are dealt to its `chunks` CTAs in interleaved blocks of rpp.
struct GnShape {
  int64_t n, hw, c, groups, cv, cpg;
  int rpp, threads;
  int64_t chunks;
};

GnShape gn_shape(int64_t n, int64_t hw, int64_t c, int64_t groups, int max_threads = kMaxThreads,
                 int ctas_per_sm = 2) {
  GnShape s;
  s.n = n; s.hw = hw; s.c = c; s.groups = groups;
  s.cv = c / 8;
  s.cpg = c / groups;
  s.rpp = (int)std::max<int64_t>(1, max_threads / s.cv);
  s.threads = (int)(s.cv * s.rpp);
  const int64_t want = std::max<int64_t>(1, (ctas_per_sm * kNumSMs + n - 1) / n);
  const int64_t blocks = (hw + s.rpp - 1) / s.rpp;          // row blocks of a sample
  s.chunks = std::min<int64_t>(want, blocks);
  return s;
}

size_t ws_bytes_for(int64_t n, int64_t hw, int64_t c, int64_t groups) {
  (void)n;
  (void)hw;
  (void)c;
  (void)groups;
  return kWsBytes;   // fixed: one workspace serves any shape (batch <= 16, groups <= 64)
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

// Per-channel fp32 sums of the CTA's rows -> row 0 of red1 / red2 (rpp rows
// folded; one thread per channel column).
__device__ __forceinline__ void fold_rows(float* red1, float* red2, int c, int rpp) {
  __syncthreads();
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
}

// ---- the statistics exchange: exact fixed-point sums, no float atomics ------
// Each producer CTA adds its per-group fp64 (sum x', sum x'^2) to the bank as
// int64 integer part + int64 2^-40 fraction (red.global.add: integer sums are
// order-independent, so the result is deterministic whichever CTA lands
// first, and no CTA waits on them).  Banks alternate per producer launch:
// launch L reads epoch e (the same for all its CTAs: e only advances after
// every CTA of L arrived), accumulates into bank e & 1, zeroes bank (e + 1) & 1
// for launch L + 1 and records cur = e & 1; its last CTA advances the epoch.
// A consumer (the apply kernel, later on the same stream) reads bank `cur`.
__device__ __forceinline__ unsigned int ld_relaxed(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

// bank of this producer launch; zeroes the idle bank (a grid-strided slice per
// CTA).  Called by every thread of the CTA (uniform control flow): ONE thread
// reads the header and shares it — every thread loading the same word would
// queue thousands of requests on one L2 address ahead of the real traffic.
__shared__ unsigned int s_snap[2];   // the producer's header snapshot (epoch, hwm)

// Producers call this right after their programmatic wait: the header read is
// then in flight during the pass instead of on its tail (nothing changes it
// before every CTA of this launch has arrived).
__device__ __forceinline__ void producer_snap(const uint8_t* ws) {
  if (threadIdx.x == 0) {
    const WsHeader* hdr = reinterpret_cast<const WsHeader*>(ws);
    s_snap[0] = ld_relaxed(&hdr->epoch);
    s_snap[1] = ld_relaxed(&hdr->hwm);
  }
}

__device__ __forceinline__ long long* producer_bank(uint8_t* ws, int nbatch, unsigned int* epoch_out = nullptr) {
  WsHeader* hdr = reinterpret_cast<WsHeader*>(ws);
  __syncthreads();                 // s_snap (producer_snap) visible
  const unsigned int epoch = s_snap[0];
  const int rows = max((int)s_snap[1], nbatch);
  if (epoch_out != nullptr) *epoch_out = epoch;
  long long* banks = reinterpret_cast<long long*>(ws + kWsHeader);
  long long* idle = banks + (size_t)((epoch + 1u) & 1u) * kBankWords;
  const int cta = blockIdx.y * gridDim.x + blockIdx.x, ctas = gridDim.x * gridDim.y;
  for (int i = cta * blockDim.x + threadIdx.x; i < rows * kMaxGroups * kGroupStride; i += ctas * blockDim.x) idle[i] = 0;
  if (cta == 0 && threadIdx.x < kMaxN)   // the resident form's counts of the next launch (any form may follow)
    reinterpret_cast<unsigned int*>(ws + kRsCntOffset)[((epoch + 1u) & 1u) * kMaxN + threadIdx.x] = 0u;
  if (cta == 0 && threadIdx.x == 0) {
    hdr->cur = epoch & 1u;
    hdr->hwm = (unsigned int)rows;
  }
  return banks + (size_t)(epoch & 1u) * kBankWords;
}

__device__ __forceinline__ void red_fixed(long long* w, double v) {
  const double hi = floor(v);
  atomicAdd(reinterpret_cast<unsigned long long*>(w), (unsigned long long)(long long)hi);
  atomicAdd(reinterpret_cast<unsigned long long*>(w + kWordPad),
            (unsigned long long)__double2ll_rn((v - hi) * kFracScale));
}
// word of moment m (0: sum, 1: sum of squares) of group g in a sample's bank
__device__ __forceinline__ long long* moment_word(long long* bank_n, int g, int m) {
  return bank_n + g * kGroupStride + 2 * m * kWordPad;
}
__device__ __forceinline__ const long long* moment_word(const long long* bank_n, int g, int m) {
  return bank_n + g * kGroupStride + 2 * m * kWordPad;
}

// this CTA is done with the bank: the last one advances the epoch
__device__ __forceinline__ void producer_arrive(uint8_t* ws) {
  __syncthreads();
  if (threadIdx.x == 0) {
    WsHeader* hdr = reinterpret_cast<WsHeader*>(ws);
    const unsigned int total = gridDim.x * gridDim.y;
    if (atomicAdd(&hdr->arrivals, 1u) == total - 1) {
      hdr->arrivals = 0u;
      atomicAdd(&hdr->epoch, 1u);
    }
  }
}

__device__ __forceinline__ double fixed_value(const long long* w) {
  return (double)__ldg(w) + (double)__ldg(w + kWordPad) / kFracScale;
}

// All index math is 32-bit within one sample (host checks n * hw * c < 2^31).
template <typename T>
__global__ void __launch_bounds__(kMaxThreads)
gn_stats_kernel(const T* __restrict__ x, const float* __restrict__ add_nc, uint8_t* __restrict__ ws, int hw, int c,
                int groups, int cpg, int rpp, int chunks) {
  pdl_wait();
  producer_snap(ws);
  extern __shared__ __align__(16) double dred[];
  double* red1 = dred;             // [rpp][c] raw sums of x
  double* red2 = dred + rpp * c;   // [rpp][c] raw sums of x^2
  const int n = blockIdx.y;
  const int cv = c >> 3;
  const int v = threadIdx.x % cv;
  const int r = threadIdx.x / cv;
  const int c0 = v * 8;
  const T* src = x + (size_t)n * hw * c + c0;
  const int step = chunks * rpp;                  // rows between this CTA's row blocks
  constexpr int U = sizeof(T) == 4 ? 2 : kStatsUnroll;   // fp32 vectors are 32 B: half as many in flight
  // shifted sums, shift = this thread's own first value per channel (no
  // cancellation, and no extra round trip for the shift)
  float2 nK[4], s1[4], s2[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) { nK[i] = s1[i] = s2[i] = f2s(0.f); }
  int mt = 0;                                     // rows this thread reduced
  for (int row0 = blockIdx.x * rpp + r; row0 < hw; row0 += U * step) {
    Raw8<T> q[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int row = row0 + u * step;
      if (row < hw) q[u] = load_raw<T>(src + (size_t)row * c);
    }
    if (mt == 0) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 k = get_pair<T>(q[0], i);
        nK[i] = make_float2(-k.x, -k.y);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (row0 + u * step < hw) {
        ++mt;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float2 d = f2add(get_pair<T>(q[u], i), nK[i]);
          s1[i] = f2add(s1[i], d);
          s2[i] = f2fma(d, d, s2[i]);
        }
      }
    }
  }
  // this thread's raw moments per channel, fp64: sum x = S1 + mt K, sum x^2 = S2 + K (2 S1 + mt K)
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const double K0 = -(double)nK[i].x, K1 = -(double)nK[i].y;
    const double a0 = s1[i].x, a1 = s1[i].y, b0 = s2[i].x, b1 = s2[i].y;
    red1[r * c + c0 + 2 * i] = a0 + mt * K0;
    red1[r * c + c0 + 2 * i + 1] = a1 + mt * K1;
    red2[r * c + c0 + 2 * i] = b0 + K0 * (2.0 * a0 + mt * K0);
    red2[r * c + c0 + 2 * i + 1] = b1 + K1 * (2.0 * a1 + mt * K1);
  }
  __syncthreads();
  if (rpp > 1) {   // fold the rpp pixel rows into row 0 (one thread per channel column)
    for (int ch = threadIdx.x; ch < c; ch += blockDim.x) {
      double a1 = red1[ch], a2 = red2[ch];
      for (int rr = 1; rr < rpp; ++rr) {
        a1 += red1[rr * c + ch];
        a2 += red2[rr * c + ch];
      }
      red1[ch] = a1;
      red2[ch] = a2;
    }
    __syncthreads();
  }
  if (add_nc != nullptr) {   // x' = x + add per channel: sum x' = sum x + m a, sum x'^2 = sum x^2 + 2 a sum x + m a^2
    int m = 0;                                    // rows this CTA reduced (per channel)
    for (int st = blockIdx.x * rpp; st < hw; st += step) m += min(rpp, hw - st);
    for (int ch = threadIdx.x; ch < c; ch += blockDim.x) {
      const double a = (double)add_nc[n * c + ch], S1 = red1[ch];
      red1[ch] = S1 + (double)m * a;
      red2[ch] = red2[ch] + a * (2.0 * S1 + (double)m * a);
    }
    __syncthreads();
  }
  // one thread per (group, moment): the group's channels in a fixed order, one
  // fixed-point red of the CTA's sum each (short independent chains; see inject_gn_kernel)
  long long* bank = producer_bank(ws, gridDim.y) + (size_t)n * kMaxGroups * kGroupStride;
  for (int v = threadIdx.x; v < 2 * groups; v += blockDim.x) {
    const double* src = (v & 1) ? red2 : red1;
    const int g = v >> 1;
    double m = 0.0;
    for (int k = 0; k < cpg; ++k) m += src[g * cpg + k];
    red_fixed(moment_word(bank, g, v & 1), m);
  }
  producer_arrive(ws);
}

constexpr int kApplyThreads = 512;
constexpr int kInjThreads = 512;

template <typename T, bool SILU>
__global__ void __launch_bounds__(kApplyThreads, 2)
gn_apply_kernel(const T* x, T* y,  // may alias: every element is read before it is written, by its own thread
                const float* __restrict__ add_nc, const uint8_t* __restrict__ ws, const float* __restrict__ gamma,
                const float* __restrict__ beta, int hw, int c, int cpg, int rpp, int chunks, float eps) {
  pdl_wait();
  const int n = blockIdx.y;
  const int cv = c >> 3;
  const int v = threadIdx.x % cv;
  const int r = threadIdx.x / cv;
  const int c0 = v * 8;
  // the group statistics from the producer's bank (fixed point -> fp64 -> mean, var)
  __shared__ float2 gstat[kMaxGroups];
  {
    const WsHeader* hdr = reinterpret_cast<const WsHeader*>(ws);
    const double count = (double)hw * (double)cpg;
    for (int g = threadIdx.x; g < c / cpg; g += blockDim.x) {
      const long long* bank = reinterpret_cast<const long long*>(ws + kWsHeader) +
                              (size_t)__ldg(&hdr->cur) * kBankWords + (size_t)n * kMaxGroups * kGroupStride;
      const double mean = fixed_value(moment_word(bank, g, 0)) / count;
      const double var = fixed_value(moment_word(bank, g, 1)) / count - mean * mean;
      gstat[g] = make_float2((float)mean, (float)(var < 0.0 ? 0.0 : var));
    }
  }
  __syncthreads();
  // this thread's 8 channels: a_c = gamma_c rstd_g, b_c = beta_c + (add_c - mean_g) a_c
  int g8[8];
  channel_groups(c0, cpg, g8);
  float2 st[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) st[j] = gstat[g8[j]];
  const float4 one = make_float4(1.f, 1.f, 1.f, 1.f), zero = make_float4(0.f, 0.f, 0.f, 0.f);
  const float4 ga0 = gamma ? *reinterpret_cast<const float4*>(gamma + c0) : one;
  const float4 ga1 = gamma ? *reinterpret_cast<const float4*>(gamma + c0 + 4) : one;
  const float4 be0 = beta ? *reinterpret_cast<const float4*>(beta + c0) : zero;
  const float4 be1 = beta ? *reinterpret_cast<const float4*>(beta + c0 + 4) : zero;
  const float4 ad0 = add_nc ? *reinterpret_cast<const float4*>(add_nc + n * c + c0) : zero;
  const float4 ad1 = add_nc ? *reinterpret_cast<const float4*>(add_nc + n * c + c0 + 4) : zero;
  const float ga[8] = {ga0.x, ga0.y, ga0.z, ga0.w, ga1.x, ga1.y, ga1.z, ga1.w};
  const float be[8] = {be0.x, be0.y, be0.z, be0.w, be1.x, be1.y, be1.z, be1.w};
  const float ad[8] = {ad0.x, ad0.y, ad0.z, ad0.w, ad1.x, ad1.y, ad1.z, ad1.w};
  float2 A[4], B[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float av[2], bv[2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int j = 2 * i + e;
      const float rstd = 1.f / sqrtf(st[j].y + eps);
      av[e] = ga[j] * rstd;
      bv[e] = be[j] + (ad[j] - st[j].x) * av[e];
      if (SILU && sizeof(T) != 4) {   // the 16-bit SiLU path works on -w (silu2_neg)
        av[e] = -av[e];
        bv[e] = -bv[e];
      }
    }
    A[i] = make_float2(av[0], av[1]);
    B[i] = make_float2(bv[0], bv[1]);
  }
  const size_t base = (size_t)n * hw * c + c0;
  const int step = chunks * rpp;
  for (int row0 = blockIdx.x * rpp + r; row0 < hw; row0 += kApplyUnroll * step) {
    Raw8<T> q[kApplyUnroll];
#pragma unroll
    for (int u = 0; u < kApplyUnroll; ++u) {
      const int row = row0 + u * step;
      if (row < hw) q[u] = load_raw<T>(x + base + (size_t)row * c);
    }
#pragma unroll
    for (int u = 0; u < kApplyUnroll; ++u) {
      const int row = row0 + u * step;
      if (row >= hw) continue;
      Raw8<T> o;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        float2 w = f2fma(get_pair<T>(q[u], i), A[i], B[i]);
        if (SILU && sizeof(T) == 4) {   // fp32 parity mode: libdevice expf + IEEE division
          w = make_float2(w.x / (1.f + expf(-w.x)), w.y / (1.f + expf(-w.y)));
        } else if (SILU) {   // SiLU(w) = w / (1 + 2^(-w log2 e)) -> 0 as w -> -inf; here w holds -w
          w = silu2_neg(w);
        }
        set_pair<T>(o, i, w);
      }
      store_raw<T>(y + base + (size_t)row * c, o);
    }
  }
}

// ---- resident form: the whole map in the SMs' shared memory, ONE launch ----
// The two-pass form pays two launch ramps and a dependent round trip per map
// (stats, then apply); at SDXL's two-pass sites those, not bytes, set its
// time.  Here one CTA per SM (a co-resident grid: cooperative launch) owns a
// contiguous run of P pixels of one sample — in NHWC one contiguous span, so
// it arrives as a few 1-D bulk copies (TMA engine, one mbarrier each) while
// the threads fold the chunks that have landed into shifted sums (one shift
// per group).  The per-group CTA partials go to the site's fixed-point bank
// (red.global.add of exact integers: deterministic in any arrival order);
// each CTA then release-adds its sample's arrival count and waits for its
// sample's CTAs only, reads the sample's statistics, applies the affine +
// SiLU to its resident tile and stores it: one read and one write of the
// map, the minimum.  Eligible while the map fits 148 tiles of <= 176 KB
// (SDXL's [2, 320, 128, 128] = 21 MB: 142 KB per CTA).
constexpr int kRsThreads = 1024;   // the largest thread count (smem / plan bounds); rs_threads() picks the launch's
constexpr int kRsMaxGroups = 32;
constexpr int kRsMaxChunks = 12;
constexpr int kRsTileMax = 176 * 1024;
constexpr int kRsExtra = kRsThreads * 4 * 8 + 2 * kRsMaxGroups * 4 + kRsMaxChunks * 8 + 4 * 4 + 128;

__device__ __forceinline__ unsigned int ld_acquire(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// a bank entry written during THIS launch: read through L2, never the
// non-coherent path
__device__ __forceinline__ double fixed_value_cg(const long long* w) {
  return (double)__ldcg(w) + (double)__ldcg(w + kWordPad) / kFracScale;
}

#ifdef SDB_RS_TRACE   // probe build only: per-CTA phase timestamps (scripts/k2r_trace.py)
__device__ unsigned long long g_rs_trace[1024][16];
#define RS_T(k)                                                          \
  if (threadIdx.x == 0) {                                                \
    g_rs_trace[blockIdx.x][k] = global_ns();                             \
    if (k == 0) {                                                        \
      unsigned int sm;                                                   \
      asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));                    \
      g_rs_trace[blockIdx.x][15] = sm;                                    \
    }                                                                    \
  }
#else
#define RS_T(k)
#endif

template <bool SILU, int NT>
__global__ void __launch_bounds__(NT, 1)
gn_resident_kernel(const __nv_bfloat16* __restrict__ x, __nv_bfloat16* __restrict__ y,
                   const float* __restrict__ gamma, const float* __restrict__ beta, const float* __restrict__ add_nc,
                   uint8_t* __restrict__ ws, int hw, int c, int cpg, int P, int per_sample, int cr, float eps) {
  extern __shared__ __align__(128) uint8_t smem[];
  RS_T(0)
  const int tid = threadIdx.x;
  const int n = blockIdx.x / per_sample;
  const int r0 = (blockIdx.x % per_sample) * P;
  const int rows = min(P, hw - r0);
  const int rowb = c * 2;
  const int nch = (rows + cr - 1) / cr;
  uint8_t* tile = smem;
  double* part = reinterpret_cast<double*>(smem + (((size_t)P * rowb + 127) & ~(size_t)127));   // [threads][4]
  float* stat = reinterpret_cast<float*>(part + NT * 4);                                  // mean | var
  uint64_t* mbar = reinterpret_cast<uint64_t*>(stat + 2 * kRsMaxGroups);
  unsigned int* snap = reinterpret_cast<unsigned int*>(mbar + kRsMaxChunks);                     // epoch, hwm, bar word
  if (tid == 0) {
    for (int k = 0; k < nch; ++k) mbar_init(smem_u32(mbar + k), 1);
    mbar_fence_init();
  }
  __syncthreads();
  pdl_wait();
  RS_T(1)
  WsHeader* hdr = reinterpret_cast<WsHeader*>(ws);
  unsigned int* cnts = reinterpret_cast<unsigned int*>(ws + kRsCntOffset);   // [2][kMaxN]
  if (tid == 0) {
    const __nv_bfloat16* xs = x + ((size_t)n * hw + r0) * c;
    const uint64_t pol = policy_evict_first();       // x is dead after this op
    for (int k = 0; k < nch; ++k) {
      const uint32_t bytes = (uint32_t)(min(cr, rows - k * cr) * rowb);
      const uint32_t bar = smem_u32(mbar + k);
      mbar_expect_tx(bar, bytes);
      bulk_g2s(smem_u32(tile + (size_t)k * cr * rowb), xs + (size_t)k * cr * c, bytes, bar, pol);
    }
  } else if (tid == 32) {   // the header, read once per CTA while the copies fly
    const unsigned int e = ld_relaxed(&hdr->epoch);
    const unsigned int hwm = ld_relaxed(&hdr->hwm);
    snap[0] = e;
    snap[1] = hwm;
    // the last CTA to have read the epoch advances it for the next launch on
    // this workspace (every CTA of this one holds e by then); no CTA waits
    if (atomicAdd(&hdr->arrivals, 1u) == gridDim.x - 1u) {
      hdr->arrivals = 0u;
      hdr->cur = e & 1u;
      hdr->hwm = (unsigned int)max((int)hwm, (int)(gridDim.x / per_sample));
      hdr->epoch = e + 1u;
    }
  }

  const int cv = c >> 3;
  const int rstep = NT / cv;
  const int j = tid % cv;
  const int rstart = tid / cv;
  const bool active = rstart < rstep;
  const int ch0 = j * 8;
  const int gA = ch0 / cpg;
  const int nA = min(8, (gA + 1) * cpg - ch0);        // leading elements in group gA, the rest in gA + 1
  const int gs = c / cpg;
  // this thread's per-(n, c) add, loaded while the copies fly
  const float* addp = add_nc != nullptr ? add_nc + (size_t)n * c + ch0 : nullptr;
  float ad[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) ad[e] = addp != nullptr ? __ldg(addp + e) : 0.f;

  // ---- statistics, chunk by chunk as the copies land ------------------------
  // Shifted sums with ONE shift per group, K_g = x[first pixel of this CTA,
  // first channel of g]: every thread of the CTA uses the same shift for a
  // group, so the per-thread fp32 sums add up directly (no cancellation, no
  // fp64 until one value per group — dependent fp64 chains are slow here).
  mbar_wait(smem_u32(mbar), 0);
  const int gB = min(gA + 1, gs - 1);
  const float KA = __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(tile)[gA * cpg]);
  const float KB = __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(tile)[gB * cpg]);
  float Kp[8], s1[8], s2[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    Kp[e] = (e < nA ? KA : KB) - ad[e];     // d = x + add - K_g
    s1[e] = s2[e] = 0.f;
  }
  for (int k = 0; k < nch; ++k) {
    mbar_wait(smem_u32(mbar + k), 0);
    if (!active) continue;
    const int rend = min(rows, (k + 1) * cr);
    for (int r = k * cr + rstart; r < rend; r += rstep) {
      const uint4 u = *reinterpret_cast<const uint4*>(tile + (size_t)r * rowb + ch0 * 2);
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float2 f = __bfloat1622float2(h[q]);
        const float d0 = f.x - Kp[2 * q], d1 = f.y - Kp[2 * q + 1];
        s1[2 * q] += d0;
        s1[2 * q + 1] += d1;
        s2[2 * q] = fmaf(d0, d0, s2[2 * q]);
        s2[2 * q + 1] = fmaf(d1, d1, s2[2 * q + 1]);
      }
    }
  }
  RS_T(2)
  {  // this thread's shifted sums collapsed onto the (<= 2) groups of its column
    float a1 = 0.f, a2 = 0.f, b1 = 0.f, b2 = 0.f;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      if (e < nA) { a1 += s1[e]; a2 += s2[e]; }
      else { b1 += s1[e]; b2 += s2[e]; }
    }
    reinterpret_cast<float4*>(part)[tid] = active ? make_float4(a1, a2, b1, b2) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  __syncthreads();
  RS_T(6)
  const unsigned int e0 = snap[0];
  long long* banks = reinterpret_cast<long long*>(ws + kWsHeader);
  long long* bank = banks + (size_t)(e0 & 1u) * kBankWords + (size_t)n * kMaxGroups * kGroupStride;
  // two short, fixed-order stages (a warp per group walked its columns and
  // shuffled serially: ~3 us of dependent latency at 4 warps per scheduler):
  //   1. column sums: one thread per (column, component) over the rstep rows
  //   2. group sums: one thread per (group, moment) over its <= 3 columns,
  //      fp64 raw moments, one fixed-point red each
  float4* part4 = reinterpret_cast<float4*>(part);
  float* colsum = reinterpret_cast<float*>(part4 + NT);          // [cv][4]
  for (int v = tid; v < cv * 4; v += NT) {
    const int col = v >> 2, comp = v & 3;
    const float* src = reinterpret_cast<const float*>(part4 + col) + comp;
    float acc = 0.f;
    for (int q = 0; q < rstep; ++q) acc += src[q * cv * 4];
    colsum[v] = acc;
  }
  __syncthreads();
  for (int v = tid; v < gs * 2; v += NT) {
    const int g = v >> 1, mom = v & 1;
    const int jlo = (g * cpg) >> 3, jhi = min(cv - 1, ((g + 1) * cpg - 1) >> 3);
    float m1 = 0.f, m2 = 0.f;
    for (int jj = jlo; jj <= jhi; ++jj) {
      const int off = jj * 8 >= g * cpg ? 0 : 2;        // the column's A part starts in it, else its B part
      m1 += colsum[jj * 4 + off];
      m2 += colsum[jj * 4 + off + 1];
    }
    // raw moments of x' over this CTA's rows x cpg channels of the group, in fp64
    const double K = (double)__bfloat162float(reinterpret_cast<const __nv_bfloat16*>(tile)[g * cpg]);
    const double M = (double)rows * cpg, S1 = m1;
    red_fixed(moment_word(bank, g, mom), mom == 0 ? S1 + M * K : (double)m2 + K * (2.0 * S1 + M * K));
  }
  // ---- per-sample completion: one release-add per CTA on its sample's count
  __syncthreads();                                   // every group's reds issued
  RS_T(3)
  unsigned int* cnt = cnts + (e0 & 1u) * kMaxN + n;
  if (tid == 0) asm volatile("fence.acq_rel.gpu;\n\tred.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(cnt) : "memory");
  {  // zero the idle bank and counts for the next producer launch on this workspace (a slice per CTA)
    const int brows = max((int)snap[1], (int)(gridDim.x / per_sample));
    long long* idle = banks + (size_t)((e0 + 1u) & 1u) * kBankWords;
    for (int i = blockIdx.x * NT + tid; i < brows * kMaxGroups * kGroupStride; i += gridDim.x * NT) idle[i] = 0;
    if (blockIdx.x == 0 && tid < kMaxN) cnts[((e0 + 1u) & 1u) * kMaxN + tid] = 0u;
  }
  float ga[8], be[8];   // the affine parameters, in flight across the barrier
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    ga[e] = gamma != nullptr ? __ldg(gamma + ch0 + e) : 1.f;
    be[e] = beta != nullptr ? __ldg(beta + ch0 + e) : 0.f;
  }
  if (tid < gs) {
    // the sample's statistics are final once all its CTAs have counted in;
    // co-residency is guaranteed by the cooperative launch, and the watchdog
    // turns a broken guarantee into a loud fault instead of a hung GPU
    const unsigned long long t0 = global_ns();
    while (ld_acquire(cnt) < (unsigned int)per_sample) {
      if (global_ns() - t0 > 2000000000ull) __trap();
    }
    const double count = (double)hw * cpg;
    const double mean = fixed_value_cg(moment_word(bank, tid, 0)) / count;
    double var = fixed_value_cg(moment_word(bank, tid, 1)) / count - mean * mean;
    var = var < 0.0 ? 0.0 : var;
    stat[tid] = (float)mean;
    stat[kRsMaxGroups + tid] = (float)var;
  }
  __syncthreads();
  RS_T(4)
  // ---- apply (+ SiLU) from shared memory, 16-B stores ------------------------
  if (!active) return;
  float2 A[4], B[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float av[2], bv[2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int ee = 2 * i + e;
      const int g = ee < nA ? gA : gA + 1;
      const float rstd = 1.f / sqrtf(stat[kRsMaxGroups + g] + eps);
      av[e] = ga[ee] * rstd;
      bv[e] = be[ee] + (ad[ee] - stat[g]) * av[e];
      if (SILU) {   // silu2_neg works on -w
        av[e] = -av[e];
        bv[e] = -bv[e];
      }
    }
    A[i] = make_float2(av[0], av[1]);
    B[i] = make_float2(bv[0], bv[1]);
  }
  __nv_bfloat16* ys = y + ((size_t)n * hw + r0) * c + ch0;
  for (int r = rstart; r < rows; r += rstep) {
    Raw8<__nv_bfloat16> q;
    q.u = *reinterpret_cast<const uint4*>(tile + (size_t)r * rowb + ch0 * 2);
    Raw8<__nv_bfloat16> o;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float2 w = f2fma(get_pair<__nv_bfloat16>(q, i), A[i], B[i]);
      if (SILU) w = silu2_neg(w);   // as gn_apply_kernel (w holds -w here)
      set_pair<__nv_bfloat16>(o, i, w);
    }
    store_raw<__nv_bfloat16>(ys + (size_t)r * c, o);
  }
  RS_T(5)
}

struct RsPlan {
  int P = 0, per_sample = 0, cr = 0, ctas = 0;
  size_t smem = 0;
};

// threads per CTA: SDB_GN_RS_THREADS = 512 (default, measured best) / 768 / 1024 (probe knob)
int rs_threads() {
  static int nt = -1;
  if (nt < 0) {
    nt = 512;
    if (const char* e = getenv("SDB_GN_RS_THREADS")) nt = atoi(e);
    if (nt != 768 && nt != 1024) nt = 512;
  }
  return nt;
}

// SMs a cooperative grid may span on the current device (0: no cooperative launch)
int rs_coop_sms() {
  static int sms = -1;
  if (sms < 0) {
    int dev = 0, coop = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) sms = 0;
    cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
    if (!coop) sms = 0;
    cudaGetLastError();
  }
  return sms;
}

bool rs_plan(int64_t n, int64_t hw, int64_t c, int64_t groups, RsPlan& p) {
  const int64_t cpg = c / groups;
  const int nt = rs_threads();
  if (groups > kRsMaxGroups || c % 8 != 0 || c / 8 > nt) return false;
  if (cpg < 8) return false;                        // an 8-channel vector spans <= 2 groups
  if (n > kNumSMs) return false;
  const int64_t per = kNumSMs / n;                  // CTAs per sample, one per SM
  int64_t P = (hw + per - 1) / per;
  if (P * c * 2 > kRsTileMax) return false;
  const int64_t per_sample = (hw + P - 1) / P;      // every CTA owns >= 1 row
  const int64_t rstep = nt / (c / 8);
  // chunks: a whole number of thread row-steps, ~8 of them per tile
  int64_t cr = std::max<int64_t>(1, (P + 7) / 8);
  cr = ((cr + rstep - 1) / rstep) * rstep;
  if ((P + cr - 1) / cr > kRsMaxChunks) return false;
  p.P = (int)P;
  p.per_sample = (int)per_sample;
  p.cr = (int)cr;
  p.ctas = (int)(n * per_sample);
  p.smem = (((size_t)P * c * 2 + 127) & ~(size_t)127) + kRsExtra;
  return true;
}

// ---- K3 + GroupNorm statistics in one pass ---------------------------------
// The input of 29 of SDXL's 46 GN sites is written by K3 (a ResNet / attention
// block's residual add, the up-block concat, a folded conv bias).  This
// kernel IS that K3 pass — out = [hidden (+hb) | skip (+sb) + sum s_i res_i] —
// and publishes the GroupNorm statistics of the rounded output into the GN
// site's workspace (the fixed-point bank, as gn_stats_kernel), so that site
// runs gn_apply_kernel alone: one full read of
// the feature map and one launch less per site.  Per thread the sums are raw
// fp32 over <= ~30 rows (relative error ~1e-6 of sum x^2, i.e. a variance
// error ~1e-6 (1 + mean^2/var) — the UNet's post-residual activations sit at
// |mean| / std = O(1); the two-pass gn_stats_kernel keeps shifted sums for
// arbitrary inputs).  Loads of a row batch are all issued before any store
// (out may alias skip).
constexpr int kInjMaxRes = 4;
template <typename T>
struct InjArgs {
  const T* res[kInjMaxRes];
  float scale[kInjMaxRes];
};

template <typename T, int NR, int KB>
__global__ void __launch_bounds__(kInjThreads)
inject_gn_kernel(T* out, const T* __restrict__ hidden, const T* skip, InjArgs<T> ra, const float* __restrict__ hb,
                 const float* __restrict__ sb, uint8_t* __restrict__ ws, int hw, int ch, int cs, int groups, int cpg,
                 int rpp, int chunks) {
  pdl_wait();
  producer_snap(ws);
  extern __shared__ __align__(16) float red[];
  const int c = ch + cs;
  float* red1 = red;               // [rpp][c]
  float* red2 = red + rpp * c;     // [rpp][c]
  const int n = blockIdx.y;
  const int cv = c >> 3, vh = ch >> 3;
  const int v = threadIdx.x % cv;
  const int r = threadIdx.x / cv;
  const int c0 = v * 8;
  const int p0 = n * hw;                           // first pixel of the sample (global pixel index)
  const int step = chunks * rpp;

  constexpr int kB = KB;
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
  for (int row0 = blockIdx.x * rpp + r; row0 < hw; row0 += kB * step) {
    Raw8<T> q0[kB], qr[kB][NR > 0 ? NR : 1];
#pragma unroll
    for (int b = 0; b < kB; ++b) {
      const int row = row0 + b * step;
      if (row < hw) {
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
      const int row = row0 + b * step;
      if (row < hw) {
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
  fold_rows(red1, red2, c, rpp);
  // one thread per (group, moment): its channels in a fixed order (fp64), one
  // fixed-point red each.  (A warp per group walking its channels and then
  // shuffling — 32 groups over the CTA's ~7 warps — chained ~5 dependent fp64
  // reductions per warp: ~10 us of tail, more than the pass itself,
  // scripts/k3_probe.py.)
  long long* bank = producer_bank(ws, gridDim.y) + (size_t)n * kMaxGroups * kGroupStride;
  for (int v = threadIdx.x; v < 2 * groups; v += blockDim.x) {
    const float* src = (v & 1) ? red2 : red1;
    const int g = v >> 1;
    double m = 0.0;
    for (int k = 0; k < cpg; ++k) m += (double)src[g * cpg + k];
    red_fixed(moment_word(bank, g, v & 1), m);
  }
  producer_arrive(ws);
}

template <typename K>
void smem_attr(K* kernel, size_t bytes) {
  if (bytes > 48 * 1024) cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

template <typename T>
int run_apply(const T* x, T* y, const float* gamma, const float* beta, const float* add_nc, const GnShape& st,
              float eps, int silu, const uint8_t* ws, cudaStream_t stream) {
  // ~4 CTAs of ~256 threads per SM (a whole number of pixel rows; up to 512
  // for the widest maps): many vectors in flight, a short a/b-table prologue
  static int knob_t = -1, knob_c = -1;     // SDB_GN_APPLY="threads,ctas_per_sm" (probe knob)
  if (knob_t < 0) {
    knob_t = 256;       // measured best (scripts/micro/k2sweep.sh): 4 CTAs of ~256 threads per SM
    knob_c = 4;
    if (const char* e = getenv("SDB_GN_APPLY")) sscanf(e, "%d,%d", &knob_t, &knob_c);
  }
  const GnShape s = gn_shape(st.n, st.hw, st.c, st.groups, knob_t, knob_c);
  if (s.threads > kApplyThreads) return fail(SDB_EINVAL, "groupnorm: channels > 4096 unsupported by the apply kernel");
  dim3 grid((unsigned)s.chunks, (unsigned)s.n);
  const size_t smem = 0;
  const int ihw = (int)s.hw, ic = (int)s.c, icpg = (int)s.cpg, ich = (int)s.chunks;
  if (silu) {
    smem_attr(gn_apply_kernel<T, true>, smem);
    launch_k(gn_apply_kernel<T, true>, grid, s.threads, smem, stream, x, y, add_nc, ws, gamma, beta, ihw, ic, icpg, s.rpp,
                                                                ich, eps);
  } else {
    smem_attr(gn_apply_kernel<T, false>, smem);
    launch_k(gn_apply_kernel<T, false>, grid, s.threads, smem, stream, x, y, add_nc, ws, gamma, beta, ihw, ic, icpg, s.rpp,
                                                                 ich, eps);
  }
  return check_launch("gn_apply_kernel");
}

template <typename T>
int run_gn(const void* xv, void* yv, const float* gamma, const float* beta, const float* add_nc, int64_t n,
           int64_t hw, int64_t c, int64_t groups, float eps, int silu, void* wsv, cudaStream_t st, bool stats) {
  const T* x = static_cast<const T*>(xv);
  T* y = static_cast<T*>(yv);
  uint8_t* ws = static_cast<uint8_t*>(wsv);
  const GnShape s = gn_shape(n, hw, c, groups);
  if (stats) {
    dim3 grid((unsigned)s.chunks, (unsigned)n);
    // (the statistics kernel's decomposition is fixed: the workspace is sized for it)
    const size_t smem = (size_t)s.rpp * c * 2 * sizeof(double);
    smem_attr(gn_stats_kernel<T>, smem);
    launch_k(gn_stats_kernel<T>, grid, s.threads, smem, st, x, add_nc, ws, (int)hw, (int)c, (int)groups, (int)s.cpg,
                                                      s.rpp, (int)s.chunks);
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
  // KB row batches of (1 + n_res) vectors in flight per thread, ~CPS CTAs of
  // ~THR threads per SM.  Measured (scripts/k3_probe.py, [2,320,128,128] + 1
  // residual): 4 / 2 / 256 (round 1) 19.8 us, 1 / 2 / 512 14.8 us; without a
  // residual 2 / 2 / 512 (11.2 us) wins.  SDB_K3GN="kb,cps,threads" overrides.
  static int env_kb = -1, env_cps = 2, env_thr = 512;
  if (env_kb < 0) {
    env_kb = 0;
    if (const char* e = getenv("SDB_K3GN")) sscanf(e, "%d,%d,%d", &env_kb, &env_cps, &env_thr);
  }
  int kb = env_kb > 0 ? env_kb : (n_res == 0 ? 2 : 1);
  if (kb != 1 && kb != 2) kb = 4;
  const int cps = std::max(1, std::min(env_cps, 8));
  const int thr = env_thr == 256 ? 256 : 512;
  const GnShape s = gn_shape(n, hw, c, groups, thr, cps);
  const int rpp = s.rpp, threads = s.threads;
  if (threads > kInjThreads) return fail(SDB_EINVAL, "residual_inject_gn: channels > 4096 unsupported");
  const size_t smem = (size_t)2 * rpp * c * sizeof(float);
  dim3 grid((unsigned)s.chunks, (unsigned)n);
  T* o = static_cast<T*>(out);
  const T* h = static_cast<const T*>(hidden);
  const T* sk = static_cast<const T*>(skip);
  uint8_t* w = static_cast<uint8_t*>(ws);
  const int ihw = (int)hw, ich = (int)ch, ics = (int)cs, ig = (int)groups, icpg = (int)(c / groups);
  const int ichunks = (int)s.chunks;
  switch (n_res) {
#define SDB_INJ_KB(NR, KB)                                                                                      \
  smem_attr(inject_gn_kernel<T, NR, KB>, smem);                                                                 \
  launch_k(inject_gn_kernel<T, NR, KB>, grid, threads, smem, st, o, h, sk, ra, hb, sb, w, ihw, ich, ics, ig, icpg, \
           rpp, ichunks);
#define SDB_INJ(NR)                                                                                            \
  case NR:                                                                                                     \
    if (kb == 1) { SDB_INJ_KB(NR, 1) } else if (kb == 2) { SDB_INJ_KB(NR, 2) } else { SDB_INJ_KB(NR, 4) }      \
    break;
    SDB_INJ(0)
    SDB_INJ(1)
    SDB_INJ(2)
    SDB_INJ(3)
    SDB_INJ(4)
#undef SDB_INJ
#undef SDB_INJ_KB
    default: return fail(SDB_EINVAL, "residual_inject_gn: at most 4 residuals");
  }
  return check_launch("inject_gn_kernel");
}

}  // namespace

size_t groupnorm_workspace(int64_t n, int64_t hw, int64_t c, int64_t groups) {
  return ws_bytes_for(n, hw, c, groups);
}

static int gn_checks(const void* x, const void* y, int64_t n, int64_t hw, int64_t c, int64_t groups, const void* ws) {
  if (n <= 0 || hw <= 0 || c <= 0 || groups <= 0) return fail(SDB_EINVAL, "groupnorm: empty shape");
  if (n > kMaxN) return fail(SDB_EINVAL, "groupnorm: batch > 16 unsupported");
  if (c % groups != 0) return fail(SDB_EINVAL, "groupnorm: channels not divisible by groups");
  if (groups > kMaxGroups) return fail(SDB_EINVAL, "groupnorm: more than 64 groups");
  if (c % 8 != 0) return fail(SDB_EINVAL, "groupnorm: channels must be a multiple of 8");
  if (c / 8 > kApplyThreads) return fail(SDB_EINVAL, "groupnorm: channels > 4096 unsupported");
  if (n * hw * c >= (int64_t)INT32_MAX - 8 * c)
    return fail(SDB_EINVAL, "groupnorm: the batch must hold < 2^31 elements");
  if (((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y)) & 15) != 0)
    return fail(SDB_EINVAL, "groupnorm: x and y must be 16-byte aligned");
  if (ws == nullptr) return fail(SDB_EINVAL, "groupnorm: workspace is NULL");
  if ((reinterpret_cast<uintptr_t>(ws) & 15) != 0) return fail(SDB_EINVAL, "groupnorm: workspace must be 16-byte aligned");
  return SDB_OK;
}

static int gn_param_checks(const float* gamma, const float* beta, const float* add_nc) {
  if (((reinterpret_cast<uintptr_t>(gamma) | reinterpret_cast<uintptr_t>(beta) |
        reinterpret_cast<uintptr_t>(add_nc)) & 15) != 0)
    return fail(SDB_EINVAL, "groupnorm: gamma / beta / add_nc must be 16-byte aligned");
  return SDB_OK;
}

int gn_cluster_try(const void* x, void* y, const float* gamma, const float* beta, const float* add_nc, int64_t n,
                   int64_t hw, int64_t c, int64_t groups, float eps, int silu, int dtype, cudaStream_t st,
                   bool* launched);

extern int g_gn_cluster_mode;   // gn_cluster.cu: 0 auto, 1 two-pass, 2 / 3 cluster forms, 4 resident form

// Auto choice of the resident form (scripts/k2_resident.py, profiles/r02_k2_resident.txt):
// wherever it is eligible — since the two-stage fold it beats the cluster
// forms at every SDXL size too ([2,640,64,64] 12.4 vs 14.2 us, [2,1280,32,32]
// 10.0 vs 12.3, [2,640,32,32] 8.3 vs 10.1); SDB_GN_RESIDENT=0 turns it off.
static bool g_rs_refused = false;   // the context refused a cooperative launch once: never try again

bool gn_resident_auto(int64_t n, int64_t hw, int64_t c, int64_t groups, int silu, int dtype) {
  if (g_rs_refused) return false;
  static int env = -1;
  if (env < 0) {
    const char* e = getenv("SDB_GN_RESIDENT");
    env = (e != nullptr && e[0] == '0') ? 0 : 1;
  }
  const int mode = g_gn_cluster_mode;
  if (dtype != SDB_BF16 || (mode != 0 && mode != 4)) return false;
  RsPlan p;
  if (!rs_plan(n, hw, c, groups, p) || p.ctas > rs_coop_sms()) return false;
  (void)silu;
  return mode == 4 || env != 0;
}

// The resident form where the shape and the device allow it; *launched tells.
static int gn_resident_try(const void* x, void* y, const float* gamma, const float* beta, const float* add_nc,
                           int64_t n, int64_t hw, int64_t c, int64_t groups, float eps, int silu, int dtype, void* ws,
                           cudaStream_t st, bool* launched) {
  *launched = false;
  if (!gn_resident_auto(n, hw, c, groups, silu, dtype)) return SDB_OK;
  RsPlan p;
  if (!rs_plan(n, hw, c, groups, p)) return SDB_OK;
  const int nt = rs_threads();
  auto kern = nt == 512   ? (silu ? gn_resident_kernel<true, 512> : gn_resident_kernel<false, 512>)
              : nt == 768 ? (silu ? gn_resident_kernel<true, 768> : gn_resident_kernel<false, 768>)
                          : (silu ? gn_resident_kernel<true, 1024> : gn_resident_kernel<false, 1024>);
  static bool attr[6] = {false, false, false, false, false, false};
  const int ai = (silu ? 1 : 0) + (nt == 512 ? 2 : nt == 768 ? 4 : 0);
  if (!attr[ai]) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)((kRsTileMax + 127) / 128 * 128 + kRsExtra));
    attr[ai] = true;
  }
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, nt, p.smem) != cudaSuccess || occ < 1) {
    cudaGetLastError();
    return SDB_OK;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)p.ctas, 1, 1);
  cfg.blockDim = dim3((unsigned)nt, 1, 1);
  cfg.dynamicSmemBytes = p.smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeCooperative;      // the grid barrier needs every CTA resident
  at[0].val.cooperative = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = g_pdl ? 2 : 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, static_cast<const __nv_bfloat16*>(x),
                                           static_cast<__nv_bfloat16*>(y), gamma, beta, add_nc,
                                           static_cast<uint8_t*>(ws), (int)hw, (int)c, (int)(c / groups), p.P,
                                           p.per_sample, p.cr, eps);
  if (e == cudaErrorCooperativeLaunchTooLarge || e == cudaErrorNotSupported || e == cudaErrorNotPermitted) {
    // a context that refuses cooperative launches (e.g. shared through MPS):
    // nothing was launched; this and every later call take the other forms
    cudaGetLastError();
    g_rs_refused = true;
    return SDB_OK;
  }
  *launched = true;
  return check_launch("gn_resident_kernel");
}

#ifdef SDB_RS_TRACE
extern "C" __attribute__((visibility("default"))) int sdb_debug_rs_trace(unsigned long long* host, int ctas) {
  return cudaMemcpyFromSymbol(host, g_rs_trace, (size_t)ctas * 16 * sizeof(unsigned long long)) == cudaSuccess ? 0 : -2;
}
#endif

// The resident form's plan for a shape (probes / tests): rows per CTA, CTAs
// per sample, chunk rows, CTAs; returns 0 when not eligible.
int gn_resident_plan(int64_t n, int64_t hw, int64_t c, int64_t groups, int* out4) {
  RsPlan p;
  if (!rs_plan(n, hw, c, groups, p)) return 0;
  const int v[4] = {p.P, p.per_sample, p.cr, p.ctas};
  for (int i = 0; i < 4; ++i) out4[i] = v[i];
  return 1;
}

int groupnorm_silu(const void* x, void* y, const float* gamma, const float* beta, const float* add_nc, int64_t n,
                   int64_t hw, int64_t c, int64_t groups, float eps, int silu, int dtype, void* ws,
                   cudaStream_t st, int stats) {
  if (int rc = gn_checks(x, y, n, hw, c, groups, ws)) return rc;
  if (int rc = gn_param_checks(gamma, beta, add_nc)) return rc;
  if (stats) {   // the resident single-launch form where the map fits the SMs' shared memory
    bool launched = false;
    if (int rc = gn_resident_try(x, y, gamma, beta, add_nc, n, hw, c, groups, eps, silu, dtype, ws, st, &launched))
      return rc;
    if (launched) return SDB_OK;
  }
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
