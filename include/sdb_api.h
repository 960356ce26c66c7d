/*
 * sdb_api.h — C-ABI of the B200-native SwiftDiffusion add-on hot path.
 *
 * The reference (addonsim 0.1.0, /root/reference/pkg) exposes this path only as
 * plain Python functions; there is no plugin / FFI layer to bind to.  Each entry
 * point below names the reference interface it replaces (file:line relative to
 * /root/reference/pkg/src/addonsim/).  The Python host package
 * (paper_2407_02031_b200) binds these with ctypes and keeps the reference
 * signatures verbatim on top.
 *
 * Conventions
 *   - All pointers are DEVICE pointers unless the parameter name ends in _host.
 *   - `stream` is a cudaStream_t passed as void* (0 = legacy default stream).
 *     Every launch is stream-ordered and asynchronous; nothing here synchronises
 *     the host, allocates persistent memory or frees caller memory.
 *   - Return value: 0 on success, negative SDB_E* code on failure;
 *     sdb_last_error() returns a thread-local message for the last failure.
 *   - Layouts: matrices are row-major with an explicit leading dimension
 *     (elements between consecutive rows); the column stride is always 1.
 *     Feature maps are NHWC (torch channels_last).
 */
#ifndef SDB_API_H_
#define SDB_API_H_

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

/* ---- error codes ------------------------------------------------------- */
#define SDB_OK 0
#define SDB_EINVAL -1   /* bad argument (shape, dtype, alignment)            */
#define SDB_ECUDA -2    /* a CUDA runtime call failed                         */
#define SDB_EUNSUP -3   /* combination not supported on this build / device   */

/* ---- dtypes -------------------------------------------------------------- */
#define SDB_F32 0
#define SDB_BF16 1
#define SDB_F16 2

/* Library version / build identification (host only). */
const char* sdb_version(void);
/* Thread-local message describing the most recent failure in this thread. */
const char* sdb_last_error(void);
/* 1 if a CUDA device of compute capability 10.x is visible, else 0. */
int sdb_device_ok(int device);

/* ========================================================================
 * K1 — LoRA patch / unpatch:  W_out = W_in + sign * scale * down @ up
 *
 * Replaces the arithmetic core of the reference:
 *   addonsim/lora.py:84-95   _accumulate(weight, adapter, scale, sign)
 * which merge_in_place (lora.py:98-104), unmerge_in_place (lora.py:107-114)
 * and create_and_replace (lora.py:132-144) all route through.  Same factor
 * convention as the reference: `down` is (h1 x rank), `up` is (rank x h2)
 * (lora.py:35-36).  Stacked adapters (lora.py:147-160) are passed as one job
 * whose rank is the sum of ranks, with per-adapter scales folded into `down`.
 *
 * Numerics: the rank contraction is accumulated in fp32 (SIMT FFMA, or the
 * tcgen05 tensor path for bf16 factors at rank >= 32) and added to W with one
 * rounding per element: W_out = round_w(fma(sign*scale, delta, float(W_in))).
 * Deterministic: no atomics, no split-K; reruns are bitwise identical.
 * ======================================================================== */
typedef struct sdb_lora_job {
  void* w_in;          /* h1 x h2, row stride ldw (elements), dtype w_dtype          */
  void* w_out;         /* output, same shape/stride as w_in; == w_in for in-place    */
  const void* down;    /* h1 x rank, row stride ldd, dtype f_dtype                   */
  const void* up;      /* rank x h2, row stride ldu, dtype f_dtype                   */
  int64_t h1, h2;
  int64_t ldw, ldd, ldu;
  int32_t rank;
  float scale;         /* multiplied by `sign` of the launch                        */
  int64_t tile_begin;  /* filled by sdb_lora_plan(): first tile index of this job   */
} sdb_lora_job;

/* Fill jobs_host[i].tile_begin for the kernel chosen by (w_dtype, f_dtype,
 * max rank) and return the total number of tiles through *total_tiles.
 * path_out (may be NULL) receives 0 = SIMT kernel, 1 = tcgen05 kernel. */
int sdb_lora_plan(sdb_lora_job* jobs_host, int n_jobs, int w_dtype, int f_dtype,
                  int64_t* total_tiles, int* path_out);

/* Batched patch over n_jobs matrices whose job table (already planned with
 * sdb_lora_plan) lives in DEVICE memory at jobs_dev.  One launch covers every
 * job; `max_ctas` > 0 caps the grid (to leave SMs to a concurrent UNet step
 * when the patch runs on a side stream), 0 = one CTA per tile. */
int sdb_lora_patch(const sdb_lora_job* jobs_dev, int n_jobs, int64_t total_tiles,
                   int w_dtype, int f_dtype, int path, float sign, int max_ctas,
                   void* stream);

/* Single-matrix convenience wrapper (no job table; used by the Python
 * merge_in_place / unmerge_in_place / create_and_replace shims). */
int sdb_lora_patch_one(void* w_in, void* w_out, int64_t h1, int64_t h2, int64_t ldw,
                       const void* down, int64_t ldd, const void* up, int64_t ldu,
                       int32_t rank, float scale, float sign,
                       int w_dtype, int f_dtype, void* stream);

/* ---- K1 fast path for bf16 serving weights (TMA + tcgen05 / FFMA) --------
 * Factors are packed once per adapter set into the UMMA K-major
 * SWIZZLE_128B layout (A = down in 128-row tiles, B = up^T in 256-column
 * panels, rank padded to a multiple of 64; buffers 1024-B aligned).  The
 * plan is a host-built blob (TMA tensor maps for every W + job/unit tables)
 * the caller copies to device memory (128-B aligned) before launching.
 * Requirements: bf16 W with ldw % 8 == 0 and 16-B aligned rows; rank <= 256.
 * simt_rank is reserved (pass 0): the contraction is tcgen05 at every rank. */
typedef struct sdb_lora_tc_job {
  void* w_in;
  void* w_out;
  int64_t h1, h2, ldw;
  const void* a_packed;
  const void* b_packed;
  int32_t rank;
  float scale;        /* epilogue scale (sdb_lora_pack_multi_layout's epi_scale x the job's own) */
  int32_t lo_mask;    /* from sdb_lora_pack_multi_layout (0 for sdb_lora_pack): K blocks with a low part */
} sdb_lora_tc_job;

int sdb_lora_pack_bytes(int64_t h1, int64_t h2, int32_t rank, size_t* a_bytes, size_t* b_bytes);
/* Stack-and-pack from up to 8 adapters' own bf16 factor buffers (the stacked
 * set of lora.py:147-160, down' = [d_i * f32(s_i)], up' = [u_i]; packed rank =
 * sum of the sources' ranks).  Scales stay exact: the scale carried by the
 * largest share of the rank (epi_scale) is applied by the patch epilogue in
 * fp32 and its sources are packed unscaled; each other source's up rows are
 * packed as x = u * (s_i / epi_scale) split into a bf16 high part and a bf16
 * low part (an extra B-panel K-block per affected K-block, bit b of
 * lo_mask, multiplied by the same A K-block), 2^-17 relative instead of a
 * bf16 rounding of s_i * d.  Query the layout first (sizes, epi_scale,
 * lo_mask for the sdb_lora_tc_job), then pack. */
typedef struct sdb_lora_src {
  const void* down; int64_t ldd;   /* h1 x rank   */
  const void* up;   int64_t ldu;   /* rank x h2   */
  int32_t rank;
  float scale;
} sdb_lora_src;
int sdb_lora_pack_multi_layout(const sdb_lora_src* srcs_host, int n_src, int64_t h1, int64_t h2,
                               size_t* a_bytes, size_t* b_bytes, float* epi_scale, int32_t* lo_mask);
int sdb_lora_pack_multi(const sdb_lora_src* srcs_host, int n_src, int64_t h1, int64_t h2,
                        void* a_packed, void* b_packed, void* stream);
int sdb_lora_pack(const void* down, int64_t ldd, const void* up, int64_t ldu, int64_t h1, int64_t h2,
                  int32_t rank, void* a_packed, void* b_packed, void* stream);
/* blob_host == NULL: only report *needed bytes, *n_units and *kb_max. */
int sdb_lora_tc_plan(const sdb_lora_tc_job* jobs_host, int n_jobs, void* blob_host, size_t blob_bytes,
                     size_t* needed, int* n_units, int* kb_max);
int sdb_lora_tc_patch(const void* blob_dev, int n_jobs, int n_units, int kb_max, int simt_rank,
                      float sign, int max_ctas, void* stream);
/* Kernel choice for plans built after the call: 0 auto (= CTA pair, fastest
 * at every rank), 1 single CTA, 2 CTA pair (cta_group::2, B panel
 * split across the two SMs of a TPC).  Returns the previous mode.  The plan
 * records its kernel in the opaque kb_max word (kb | mode << 8). */
int sdb_lora_tc_set_mode(int mode);

/* ========================================================================
 * K2 — GroupNorm (+ optional SiLU), NHWC.
 *   x' = x + add_nc[n, c]            (add_nc may be NULL: fused ResNet temb add)
 *   y  = act( (x' - mean_g(x')) * rstd_g(x') * gamma_c + beta_c )
 * The reference models this op only as a latency multiplier
 * (addonsim/model.py:66-70 unet_opt_submultipliers[2] = 1.072; paper
 * PAPER.md:572-576).  x, y: [N, HW, C] (channels innermost), dtype `dtype`;
 * gamma, beta: fp32 [C].  `workspace` must hold sdb_groupnorm_workspace()
 * bytes (a constant, ~130 KB) and be ZERO-initialised once: it holds an epoch
 * word and two fp64 accumulator banks that the launches themselves recycle
 * (each launch zeroes the bank the previous one used), so it stays valid
 * across launches and CUDA-graph replays with any shape; calls sharing a
 * workspace must be ordered on one stream.  y may alias x.
 * ======================================================================== */
size_t sdb_groupnorm_workspace(int64_t n, int64_t hw, int64_t c, int64_t groups);
/* K2 form selection: mode 0 (default) runs the resident form wherever it
 * fits (below), else a single-pass cluster form where the shape fits (bf16,
 * C/G >= 8): one launch, one read, one write, a thread-block cluster per
 * (sample, channel slab) holding that slab of the map in shared memory —
 * round 1's form for maps <= 6 MB, the streamed form (TMA chunks overlapped
 * with the statistics, each chunk stored as soon as it is normalised) for
 * larger maps whose clusters fit one wave — else the two-pass form.
 * Mode 1 forces the two-pass form, 2 only round 1's cluster form, 3 only the
 * streamed form, 4 only the resident form.  sdb_groupnorm_launches returns the kernel launches
 * sdb_groupnorm_silu will make for a shape; sdb_groupnorm_stream_plan fills
 * out7 = {slab channels, cluster CTAs, rows per CTA, rows per chunk, chunks,
 * clusters, co-resident clusters} of the streamed form (0 = not eligible). */
void sdb_groupnorm_set_mode(int mode);
int sdb_groupnorm_launches(int64_t n, int64_t hw, int64_t c, int64_t groups, int dtype);
int sdb_groupnorm_stream_plan(int64_t n, int64_t hw, int64_t c, int64_t groups, int* out7);
/* The resident form (one cooperative launch, one CTA per SM holding a run of
 * pixels of one sample in shared memory, statistics exchanged through the
 * workspace's fixed-point bank, each CTA waiting only for its sample's
 * CTAs): auto for bf16 maps with C/G >= 8, <= 32 groups and <= 148 CTAs of
 * <= 176 KB tiles (SDB_GN_RESIDENT=0 in the environment turns it off).
 * out4 = {rows per CTA, CTAs per sample, rows per copy chunk, CTAs}; 0 = not
 * eligible. */
int sdb_groupnorm_resident_plan(int64_t n, int64_t hw, int64_t c, int64_t groups, int* out4);

/* Programmatic dependent launch (default on; SDB_PDL=0 in the environment
 * turns it off at load): the streaming kernels (K2-K7, K9, K10) launch with
 * the programmatic-stream-serialisation attribute and wait (griddepcontrol)
 * before touching their predecessor's data, so their launch overlaps the tail
 * of the previous kernel on the stream.  Returns the previous setting. */
int sdb_set_pdl(int on);
int sdb_groupnorm_silu(const void* x, void* y, const float* gamma, const float* beta,
                       const float* add_nc, int64_t n, int64_t hw, int64_t c, int64_t groups, float eps,
                       int apply_silu, int dtype, void* workspace, void* stream);
/* Apply half only: the statistics of x were accumulated into `workspace` by
 * the kernel that produced x (sdb_residual_inject_gn, same groups, ordered
 * on the same stream); one read of x, one write of y, one launch. */
int sdb_groupnorm_apply(const void* x, void* y, const float* gamma, const float* beta,
                        const float* add_nc, int64_t n, int64_t hw, int64_t c, int64_t groups,
                        float eps, int apply_silu, int dtype, void* workspace, void* stream);

/* ========================================================================
 * K3 — ControlNet residual injection fused with the up-block concat.
 *   out[p, 0:ch]        = hidden[p, :]                       (hidden may be NULL)
 *   out[p, ch:ch+cs]    = skip[p, :] + sum_i scales[i] * res_i[p, :]
 * Replaces the "outputs are added up to the skip connections and middle
 * block" step (modelled as a zero-cost sum in SPEC.md:234
 * and charged only comm_ms in addonsim/model.py:151-158).
 * With hidden == NULL and ch == 0 it is the in-place mid-block add
 * (out may alias skip).  res_ptrs_host: n_res device pointers (host array).
 * ======================================================================== */
int sdb_residual_inject(void* out, const void* hidden, const void* skip,
                        const void* const* res_ptrs_host, const float* scales_host,
                        int n_res, int64_t pixels, int64_t ch, int64_t cs,
                        int dtype, void* stream);
/* Same, plus optional fp32 per-channel biases (16-B aligned, may be NULL):
 *   out[p, 0:ch]     += hidden_bias[0:ch]
 *   out[p, ch:ch+cs] += skip_bias[0:cs]   (added before the residuals)
 * — the bias of the convolution that produced hidden / skip, folded here so
 * the conv needs no separate broadcast bias pass. */
int sdb_residual_inject_bias(void* out, const void* hidden, const void* skip,
                             const void* const* res_ptrs_host, const float* scales_host,
                             int n_res, int64_t pixels, int64_t ch, int64_t cs,
                             const float* hidden_bias, const float* skip_bias,
                             int dtype, void* stream);
/* K3 + the GroupNorm statistics of its output in the same pass: out is
 * n x hw pixels of [hidden (+hidden_bias) | skip (+skip_bias) + sum_i
 * scales[i] * res_i] (NHWC), and the per-(sample, group) moments of the
 * rounded out are accumulated into gn_workspace (a sdb_groupnorm_workspace
 * buffer) for a following sdb_groupnorm_apply of out.  n_res <= 4; bf16/fp16.
 * Used where a ResNet / attention block's residual add, the up-block concat
 * or a folded conv bias writes the next GroupNorm's input (PAPER.md:572-576:
 * the fused GN+SiLU; here its statistics pass is fused into the producer). */
int sdb_residual_inject_gn(void* out, const void* hidden, const void* skip,
                           const void* const* res_ptrs_host, const float* scales_host, int n_res,
                           int64_t n, int64_t hw, int64_t ch, int64_t cs, const float* hidden_bias,
                           const float* skip_bias, int64_t groups, void* gn_workspace, int dtype, void* stream);

/* ========================================================================
 * K7 — cross-attention against a short, step-invariant context (Lk <= 128,
 * e.g. the 77 text tokens), bf16, one pass over the queries:
 *   o[b, i, h*d:(h+1)*d] = softmax(scale * q_h[i] . k_h^T) v_h
 * q: [n, lq, heads*d] rows of stride ldq; kv: [n, lk, *] rows of stride ldkv
 * holding K at column 0 and V at column voff; o: rows of stride ldo.
 * head_dim in 8..160 (% 8); strides % 8; pointers 16-B aligned.
 * The UNet's attn2 blocks (the SDPA call of a diffusers-style
 * Attention); the reference has no attention arithmetic (latency model).
 * ======================================================================== */
int sdb_cross_attention(const void* q, int64_t ldq, const void* kv, int64_t ldkv, int64_t voff, void* o,
                        int64_t ldo, int n, int lq, int lk, int heads, int head_dim, float scale, int dtype,
                        void* stream);
/* Head dim 64: 2 (default) runs the persistent tcgen05 form (one CTA per SM
 * walking a run of 128-query tiles, Q by TMA two tiles ahead, S and O
 * double-buffered in TMEM, one query row per thread) where each CTA's run
 * spans <= 2 heads and the grid holds >= 2 waves of 128-query tiles (the
 * serving batches), else as 1; 1: the per-tile tcgen05 form for one-wave
 * grids, else mma.sync; 0: every head dim runs the mma.sync form.  Returns
 * the previous setting. */
int sdb_cross_attention_set_mode(int tcgen05);

/* K8 — self-attention, head dim 64, non-causal, bf16, flash-style on tcgen05
 * (S and PV in TMEM, online softmax one query row per thread):
 *   o[b, i, h*64:(h+1)*64] = softmax(scale * q_h[i] . k_h^T) v_h
 * qkv: [n, seq_len, *] rows of stride ldqkv holding Q | K | V (heads*64
 * columns each, the fused to_qkv GEMM output); o rows of stride ldo;
 * seq_len % 128 == 0.  The UNet's attn1 blocks (the SDPA call of a
 * diffusers-style Attention); the reference has no attention arithmetic. */
int sdb_self_attention(const void* qkv, int64_t ldqkv, void* o, int64_t ldo, int n, int seq_len, int heads,
                       int head_dim, float scale, int dtype, void* stream);

/* ========================================================================
 * Peer step handshakes (ControlNet-as-a-service over NVLink, caas.py):
 * enqueue on `stream` a wait until the 32-bit word at addr (local, IPC- or
 * peer-mapped device memory) is >= value, or a write of value to addr that
 * is ordered after every earlier store/copy of the stream (system-scope
 * fence).  Replaces the per-step transfer steps modelled as comm_ms in
 * addonsim/model.py:151-158 (orchestrator.py:621-660) with GPU-side flags.
 * ======================================================================== */
int sdb_stream_wait_value32(void* stream, void* addr, uint32_t value);
int sdb_stream_write_value32(void* stream, void* addr, uint32_t value);
/* Stream-ordered copy between any two device addresses (local, peer over
 * NVLink, or CUDA-IPC mapped): the residual push / latent pull of caas.py. */
int sdb_memcpy_async(void* dst, const void* src, size_t bytes, void* stream);

/* ========================================================================
 * K5 — GEGLU: out[m, 0:f] = proj[m, 0:f] * gelu(proj[m, f:2f]) (exact erf).
 * The paper's fused GEGLU; in the reference only the
 * 1.06 sub-multiplier of addonsim/model.py:66-70.  f % 8 == 0.
 * ======================================================================== */
int sdb_geglu(const void* proj, void* out, int64_t rows, int64_t f, int dtype, void* stream);

/* K10 — nearest 2x upsample of an NHWC map: y[n, 2i+a, 2j+b, :] = x[n, i, j, :]
 * (the UNet decoder's upsample before its 3x3 conv).  x [n, h, w, c], y
 * [n, 2h, 2w, c], c * elem_bytes a multiple of 16, 16-B aligned pointers.
 * No reference counterpart (addonsim has no UNet arithmetic). */
/* Batched copy — restore-from-pristine unpatch of every patched matrix in
 * ONE launch (the reference unmerges by subtracting, lora.py:107-114; a
 * serving copy can restore W exactly).  Device arrays: per tensor its source,
 * destination (16-B aligned), size in 16-B vectors, and the exclusive prefix
 * of its chunk counts (n + 1 entries; a chunk is
 * sdb_batched_copy_chunk_vectors() vectors). */
int64_t sdb_batched_copy_chunk_vectors(void);
int sdb_batched_copy(const void* const* src_dev, void* const* dst_dev, const int64_t* nvec_dev,
                     const int64_t* chunk_prefix_dev, int n, int64_t total_chunks, void* stream);
int sdb_upsample2x(const void* x, void* y, int64_t n, int64_t h, int64_t w, int64_t c, int elem_bytes,
                   void* stream);

/* ========================================================================
 * K6 — residual add + LayerNorm of the transformer blocks:
 *   x[m] += d[m] (in place; d may be NULL), y[m] = LN(x[m]) * gamma + beta.
 * gamma / beta in the same dtype as x; C % 8 == 0, C <= 2560.
 * ======================================================================== */
int sdb_add_layernorm(void* x, const void* d, void* y, const void* gamma, const void* beta,
                      int64_t rows, int64_t c, float eps, int dtype, void* stream);

/* K5' — the transformer FF projection with GEGLU fused into its epilogue (one
 * tcgen05 GEMM; the paper's fused GEGLU):
 *   out[m, j] = (x w_v^T + b_v)[m, j] * gelu((x w_g^T + b_g)[m, j])
 * x: [m, k] bf16 rows, w: [2f, k] bf16 (value rows, then gate rows: the GEGLU
 * proj weight as stored), bias: [2f] fp32 or NULL, out: [m, f] bf16.
 * k % 64 == 0, f % 128 == 0, 16-B aligned pointers. */
int sdb_ff_geglu(const void* x, const void* w, const float* bias, void* out, int64_t m, int64_t k, int64_t f,
                 void* stream);

/* ========================================================================
 * K4 — classifier-free guidance + DDIM (eta = 0) step, fused.
 *   eps     = eps_u + g * (eps_c - eps_u)           (eps = [eps_u ; eps_c])
 *   x0      = (x - sqrt(1 - a_t) * eps) / sqrt(a_t)
 *   x_prev  = sqrt(a_prev) * x0 + sqrt(1 - a_prev) * eps
 * writes x_prev into x_out (fp32 master latent, may alias x) and, when
 * unet_in != NULL, into both CFG halves of the next UNet input (dtype
 * `in_dtype`).  Per-step coefficients are read from the device table
 * coef[step][4] = {a_t, a_prev, guidance, unused} at index *step_dev, and
 * *step_dev is incremented by the kernel, so a whole step is graph-capturable.
 * Not in the reference at all.
 * ======================================================================== */
int sdb_cfg_ddim_step(const void* eps, int eps_dtype, const float* x, float* x_out,
                      void* unet_in, int in_dtype, int64_t latent_elems,
                      const float* coef, int* step_dev, void* stream);

/* ========================================================================
 * K9 — the UNet output convolution: 3x3, pad 1, C -> 4 channels, fp32 out.
 *   out[n, y, x, o] = bias[o] + sum_{dy, dx, c} x[n, y+dy-1, x+dx-1, c] * w[o, dy, dx, c]
 * x: NHWC (channels_last) [n, h, width, c] of `dtype` (SDB_BF16 / SDB_F32);
 * w: the weight's physical channels_last layout [cout, 3, 3, c], same dtype;
 * bias: fp32 [cout] or NULL; out: fp32 NHWC [n, h, width, cout].
 * fp32 accumulation.  cout must be 4, width a multiple of 16, c even <= 1280.
 * Replaces the UNet's conv_out (no reference counterpart: SURVEY §0.2).
 * ======================================================================== */
int sdb_conv_out(const void* x, const void* w, const float* bias, float* out, int64_t n, int64_t h,
                 int64_t width, int64_t c, int64_t cout, int dtype, void* stream);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif

#ifdef __cplusplus
}
#endif
#endif /* SDB_API_H_ */
