// lora_patch.cu — K1: batched LoRA patch / unpatch, SIMT path.
//
//   W_out[r, c] = round_w( fma(sign*scale, sum_k down[r,k] * up[k,c], float(W_in[r,c])) )
//
// Restates the arithmetic of addonsim/lora.py:84-95 (_accumulate): one
// W read-modify-write per element, the rank contraction never materialised
// as a full h1 x h2 delta, one rounding into W.  The
// reference accumulates the contraction in fp64 with numpy/OpenBLAS; here it
// is accumulated in fp32 FFMA in ascending-k order (deterministic, no
// atomics, no split-K), which keeps |W_gpu - W_ref| within one W ulp plus
// ~rank * 2^-24 * |delta| — far inside the reference's 1e-5 gates
// (tests/test_lora.py:81-101, tests/test_acceptance.py:341-391).
//
// Work decomposition: every job (one weight matrix) is cut into 64 x 128
// tiles; the tiles of all jobs form one flat index space (job.tile_begin is
// the prefix sum computed by sdb_lora_plan), so one launch patches every
// matrix of a UNet (794 for SDXL) with no per-layer launch overhead.  The
// grid is persistent-capable: a capped grid (max_ctas) strides over tiles,
// which is how the patch leaves SMs to a concurrent denoising step.
//
// Memory: the W tile is prefetched into registers (16 B vector loads) at the
// start of the tile so its HBM latency overlaps the factor loads and the
// FFMA contraction; factors are staged through shared memory in 32-deep
// k-chunks (any rank).  This kernel is HBM-bound for bf16 W at rank <= 16
// and for fp32 W at rank <= ~32; above that the tcgen05 path
// (lora_patch_tc.cu) takes bf16 jobs.
#include "common.cuh"

namespace sdb {
namespace {

constexpr int BM = 64;
constexpr int BN = 128;
constexpr int KC = 32;
constexpr int THREADS = 256;

struct TileInfo {
  const void* w_in;
  void* w_out;
  const void* down;
  const void* up;
  int64_t h1, h2, ldw, ldd, ldu;
  int64_t row0, col0;
  int rank;
  float ss;  // sign * scale
  int vec;   // 16-byte vector path legal for this job
};

template <typename TW>
__device__ __forceinline__ bool vec_ok(const void* a, const void* b, int64_t ldw) {
  constexpr int64_t kAlignElems = 16 / sizeof(TW);
  return ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b)) & 15) == 0 &&
         (ldw % kAlignElems) == 0;
}

template <typename TW, typename TF>
__global__ void __launch_bounds__(THREADS)
lora_patch_simt_kernel(const sdb_lora_job* __restrict__ jobs, const sdb_lora_job one,
                       int n_jobs, int64_t total_tiles, float sign) {
  __shared__ float sd[KC][BM + 1];             // down^T chunk (k-major), +1 pad: conflict-free stores
  __shared__ __align__(16) float su[KC][BN];   // up chunk
  __shared__ TileInfo ti;

  const int tid = threadIdx.x;
  const int tx = tid & 15;   // 8-column group
  const int ty = tid >> 4;   // row group: rows ty + 16*i

  for (int64_t tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
    if (tid == 0) {
      // jobs == nullptr: single job passed by value (sdb_lora_patch_one)
      int lo = 0, hi = n_jobs - 1;
      while (jobs != nullptr && lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (jobs[mid].tile_begin <= tile) lo = mid; else hi = mid - 1;
      }
      const sdb_lora_job& J = jobs != nullptr ? jobs[lo] : one;
      int64_t local = tile - J.tile_begin;
      int64_t tiles_n = (J.h2 + BN - 1) / BN;
      ti.w_in = J.w_in; ti.w_out = J.w_out; ti.down = J.down; ti.up = J.up;
      ti.h1 = J.h1; ti.h2 = J.h2; ti.ldw = J.ldw; ti.ldd = J.ldd; ti.ldu = J.ldu;
      ti.row0 = (local / tiles_n) * BM;
      ti.col0 = (local % tiles_n) * BN;
      ti.rank = J.rank;
      ti.ss = sign * J.scale;
      ti.vec = vec_ok<TW>(J.w_in, J.w_out, J.ldw);
    }
    __syncthreads();
    const TW* __restrict__ w_in = static_cast<const TW*>(ti.w_in);
    TW* __restrict__ w_out = static_cast<TW*>(ti.w_out);
    const TF* __restrict__ down = static_cast<const TF*>(ti.down);
    const TF* __restrict__ up = static_cast<const TF*>(ti.up);
    const int64_t h1 = ti.h1, h2 = ti.h2, ldw = ti.ldw;
    const int64_t row0 = ti.row0, col0 = ti.col0;
    const int rank = ti.rank;
    const float ss = ti.ss;
    const int64_t col = col0 + 8 * tx;
    const bool full_vec = ti.vec && (col + 8 <= h2);

    // ---- prefetch the W tile (4 rows x 8 cols per thread) -----------------
    float wv[4][8];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int64_t row = row0 + ty + 16 * i;
      if (row < h1) {
        const TW* p = w_in + row * ldw + col;
        if (full_vec) {
          Vec8<TW>::load(p, wv[i]);
        } else {
#pragma unroll
          for (int j = 0; j < 8; ++j) wv[i][j] = (col + j < h2) ? to_f32<TW>(p[j]) : 0.f;
        }
      }
    }

    // ---- rank contraction in fp32, ascending k ----------------------------
    float acc[4][8];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;

    for (int k0 = 0; k0 < rank; k0 += KC) {
      const int kc = min(KC, rank - k0);
      // down chunk: BM x kc -> sd[k][r]; up chunk: kc x BN -> su[k][c].  Fixed
      // trip counts, fully unrolled: all 24 loads of a thread are in flight
      // together (a runtime-bounded loop issued them one latency at a time —
      // 48 us for SDXL's 320 x 36 conv_in, a 5-CTA launch)
      static_assert((BM * KC) % THREADS == 0 && (KC * BN) % THREADS == 0, "even load split");
      float dv[BM * KC / THREADS], uv[KC * BN / THREADS];
#pragma unroll
      for (int i = 0; i < BM * KC / THREADS; ++i) {
        const int e = tid + i * THREADS;
        const int r = e / KC, k = e % KC;
        const int64_t row = row0 + r;
        dv[i] = (k < kc && row < h1) ? to_f32<TF>(down[row * ti.ldd + k0 + k]) : 0.f;
      }
#pragma unroll
      for (int i = 0; i < KC * BN / THREADS; ++i) {
        const int e = tid + i * THREADS;
        const int k = e / BN, c = e % BN;
        uv[i] = (k < kc && col0 + c < h2) ? to_f32<TF>(up[(int64_t)(k0 + k) * ti.ldu + col0 + c]) : 0.f;
      }
#pragma unroll
      for (int i = 0; i < BM * KC / THREADS; ++i) {
        const int e = tid + i * THREADS;
        sd[e % KC][e / KC] = dv[i];
      }
#pragma unroll
      for (int i = 0; i < KC * BN / THREADS; ++i) {
        const int e = tid + i * THREADS;
        su[e / BN][e % BN] = uv[i];
      }
      __syncthreads();
      for (int k = 0; k < kc; ++k) {
        float a[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = sd[k][ty + 16 * i];
        const float4 b0 = *reinterpret_cast<const float4*>(&su[k][8 * tx]);
        const float4 b1 = *reinterpret_cast<const float4*>(&su[k][8 * tx + 4]);
        const float b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
      }
      __syncthreads();
    }

    // ---- single-rounding update of W ---------------------------------------
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int64_t row = row0 + ty + 16 * i;
      if (row < h1) {
        float o[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) o[j] = fmaf(ss, acc[i][j], wv[i][j]);
        TW* p = w_out + row * ldw + col;
        if (full_vec) {
          Vec8<TW>::store(p, o);
        } else {
#pragma unroll
          for (int j = 0; j < 8; ++j)
            if (col + j < h2) p[j] = from_f32<TW>(o[j]);
        }
      }
    }
    __syncthreads();  // ti is rewritten by the next tile
  }
}

template <typename TW, typename TF>
int launch_simt(const sdb_lora_job* jobs_dev, const sdb_lora_job& one, int n_jobs,
                int64_t total_tiles, float sign, int max_ctas, cudaStream_t st) {
  int64_t grid = total_tiles;
  if (max_ctas > 0 && grid > max_ctas) grid = max_ctas;
  if (grid > (int64_t)1 << 30) grid = (int64_t)1 << 30;
  lora_patch_simt_kernel<TW, TF><<<(unsigned)grid, THREADS, 0, st>>>(jobs_dev, one, n_jobs, total_tiles, sign);
  return check_launch("lora_patch_simt_kernel");
}

}  // namespace

int64_t simt_tiles(int64_t h1, int64_t h2) {
  return ((h1 + BM - 1) / BM) * ((h2 + BN - 1) / BN);
}

int lora_patch_simt(const sdb_lora_job* jobs_dev, const sdb_lora_job& one, int n_jobs,
                    int64_t total_tiles, int w_dtype, int f_dtype, float sign, int max_ctas,
                    cudaStream_t st) {
  if (w_dtype == SDB_F32 && f_dtype == SDB_F32)
    return launch_simt<float, float>(jobs_dev, one, n_jobs, total_tiles, sign, max_ctas, st);
  if (w_dtype == SDB_BF16 && f_dtype == SDB_BF16)
    return launch_simt<__nv_bfloat16, __nv_bfloat16>(jobs_dev, one, n_jobs, total_tiles, sign, max_ctas, st);
  if (w_dtype == SDB_BF16 && f_dtype == SDB_F32)
    return launch_simt<__nv_bfloat16, float>(jobs_dev, one, n_jobs, total_tiles, sign, max_ctas, st);
  if (w_dtype == SDB_F16 && f_dtype == SDB_F16)
    return launch_simt<__half, __half>(jobs_dev, one, n_jobs, total_tiles, sign, max_ctas, st);
  if (w_dtype == SDB_F32 && f_dtype == SDB_BF16)
    return launch_simt<float, __nv_bfloat16>(jobs_dev, one, n_jobs, total_tiles, sign, max_ctas, st);
  return fail(SDB_EUNSUP, "lora_patch: unsupported (w_dtype, f_dtype) combination");
}

}  // namespace sdb
