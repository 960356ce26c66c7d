// api.cu — the extern "C" boundary declared in include/sdb_api.h.
// Argument validation + dispatch only; the kernels live in the other units.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>

#include "common.cuh"

namespace sdb {

thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }

// programmatic dependent launch for the streaming kernels (common.cuh); SDB_PDL=0 turns it off
static int pdl_default() {
  const char* e = getenv("SDB_PDL");
  return e == nullptr || atoi(e) != 0;
}
int g_pdl = pdl_default();

// lora_patch.cu
int64_t simt_tiles(int64_t h1, int64_t h2);
int lora_patch_simt(const sdb_lora_job* jobs_dev, const sdb_lora_job& one, int n_jobs,
                    int64_t total_tiles, int w_dtype, int f_dtype, float sign, int max_ctas,
                    cudaStream_t st);
// lora_patch_tc.cu
void tc_pack_bytes(int64_t h1, int64_t h2, int rank, size_t* a_bytes, size_t* b_bytes);
int tc_pack(const void* down, int64_t ldd, const void* up, int64_t ldu, int64_t h1, int64_t h2, int rank,
            void* a_out, void* b_out, cudaStream_t st);
int tc_pack_multi(const sdb_lora_src* srcs, int n_src, int64_t h1, int64_t h2, void* a_out, void* b_out,
                  cudaStream_t st);
int tc_pack_multi_layout(const sdb_lora_src* srcs, int n_src, int64_t h1, int64_t h2, size_t* a_bytes,
                         size_t* b_bytes, float* epi_scale, int32_t* lo_mask);
int tc_plan(const sdb_lora_tc_job* jobs, int n_jobs, void* blob, size_t blob_bytes, size_t* needed,
            int* n_units_out, int* kb_max_out);
int tc_set_mode(int mode);
int tc_patch(const void* blob_dev, int n_jobs, int n_units, int kb_max, int simt_rank, float sign,
             int max_ctas, cudaStream_t st);
// groupnorm_silu.cu
size_t groupnorm_workspace(int64_t n, int64_t hw, int64_t c, int64_t groups);
int groupnorm_silu(const void* x, void* y, const float* gamma, const float* beta,
                   const float* add_nc, int64_t n, int64_t hw, int64_t c, int64_t groups, float eps, int silu, int dtype,
                   void* ws, cudaStream_t st, int stats);
int residual_inject_gn(void* out, const void* hidden, const void* skip, const void* const* res, const float* scales,
                       int n_res, int64_t n, int64_t hw, int64_t ch, int64_t cs, const float* hidden_bias,
                       const float* skip_bias, int64_t groups, void* ws, int dtype, cudaStream_t st);
// residual_inject.cu
int residual_inject(void* out, const void* hidden, const void* skip, const void* const* res,
                    const float* scales, int n_res, int64_t pixels, int64_t ch, int64_t cs,
                    const float* hidden_bias, const float* skip_bias, int dtype, cudaStream_t st);
// fused_ops.cu
int geglu(const void* proj, void* out, int64_t rows, int64_t f, int dtype, cudaStream_t st);
int upsample2x(const void* x, void* y, int64_t n, int64_t h, int64_t w, int64_t c, int elem_bytes, cudaStream_t st);
int batched_copy(const void* const* src_dev, void* const* dst_dev, const int64_t* nvec_dev,
                 const int64_t* chunk_prefix_dev, int n, int64_t total_chunks, cudaStream_t st);
int64_t batched_copy_chunk_vectors();
int ff_geglu(const void* x, const void* w, const float* bias, void* out, int64_t m, int64_t k, int64_t f,
             cudaStream_t st);
int add_layernorm(void* x, const void* d, void* y, const void* gamma, const void* beta, int64_t rows, int64_t c,
                  float eps, int dtype, cudaStream_t st);
// cross_attn.cu
int cross_attention(const void* q, int64_t ldq, const void* kv, int64_t ldkv, int64_t voff, void* o, int64_t ldo,
                    int n, int lq, int lk, int heads, int d, float scale, int dtype, cudaStream_t st);
int cross_attention_set_mode(int tc);
// self_attn.cu
int self_attention(const void* qkv, int64_t ldqkv, void* o, int64_t ldo, int n, int L, int heads, int head_dim,
                   float scale, int dtype, cudaStream_t st);
// peer_sync.cu
int stream_wait_value32(cudaStream_t st, void* addr, uint32_t value);
int stream_write_value32(cudaStream_t st, void* addr, uint32_t value);
int memcpy_async(void* dst, const void* src, size_t bytes, cudaStream_t st);
// gn_cluster.cu
extern int g_gn_cluster_mode;
int gn_launches(int64_t n, int64_t hw, int64_t c, int64_t groups, int dtype);
int gn_stream_plan(int64_t n, int64_t hw, int64_t c, int64_t groups, int* out7);
int gn_resident_plan(int64_t n, int64_t hw, int64_t c, int64_t groups, int* out4);
// conv_out.cu
int conv_out(const void* x, const void* w, const float* bias, float* out, int64_t n, int64_t h, int64_t w_,
             int64_t c, int64_t cout, int dtype, cudaStream_t st);
// cfg_step.cu
int cfg_ddim_step(const void* eps, int eps_dtype, const float* x, float* x_out, void* unet_in,
                  int in_dtype, int64_t L, const float* coef, int* step_dev, cudaStream_t st);

static int check_job(const sdb_lora_job& j, int idx) {
  if (j.h1 <= 0 || j.h2 <= 0)
    return fail(SDB_EINVAL, "lora job " + std::to_string(idx) + ": empty weight");
  if (j.rank <= 0) return fail(SDB_EINVAL, "lora job " + std::to_string(idx) + ": rank must be >= 1");
  if (j.ldw < j.h2 || j.ldu < j.h2 || j.ldd < j.rank)
    return fail(SDB_EINVAL, "lora job " + std::to_string(idx) + ": leading dimension too small");
  if (!j.w_in || !j.w_out || !j.down || !j.up)
    return fail(SDB_EINVAL, "lora job " + std::to_string(idx) + ": NULL pointer");
  return SDB_OK;
}

}  // namespace sdb

using namespace sdb;

extern "C" {

const char* sdb_version(void) { return "sdb 0.1.0 (sm_100a)"; }

const char* sdb_last_error(void) { return g_last_error.c_str(); }

int sdb_device_ok(int device) {
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return prop.major == 10 ? 1 : 0;
}

int sdb_lora_plan(sdb_lora_job* jobs, int n_jobs, int w_dtype, int f_dtype, int64_t* total_tiles,
                  int* path_out) {
  if (n_jobs <= 0 || jobs == nullptr || total_tiles == nullptr)
    return fail(SDB_EINVAL, "sdb_lora_plan: no jobs");
  (void)w_dtype;
  (void)f_dtype;
  for (int i = 0; i < n_jobs; ++i)
    if (int rc = check_job(jobs[i], i)) return rc;
  // the job-table API runs the generic SIMT kernel (any dtype, any stride);
  // the tcgen05 path has its own packed-factor plan (sdb_lora_tc_plan)
  int64_t t = 0;
  for (int i = 0; i < n_jobs; ++i) {
    jobs[i].tile_begin = t;
    t += simt_tiles(jobs[i].h1, jobs[i].h2);
  }
  *total_tiles = t;
  if (path_out) *path_out = 0;
  return SDB_OK;
}

int sdb_lora_patch(const sdb_lora_job* jobs_dev, int n_jobs, int64_t total_tiles, int w_dtype,
                   int f_dtype, int path, float sign, int max_ctas, void* stream) {
  if (n_jobs <= 0 || jobs_dev == nullptr) return fail(SDB_EINVAL, "sdb_lora_patch: no jobs");
  if (total_tiles <= 0) return fail(SDB_EINVAL, "sdb_lora_patch: plan has no tiles");
  if (path != 0)
    return fail(SDB_EUNSUP, "sdb_lora_patch: path 1 is planned by sdb_lora_tc_plan / run by sdb_lora_tc_patch");
  sdb_lora_job none;
  std::memset(&none, 0, sizeof(none));
  return lora_patch_simt(jobs_dev, none, n_jobs, total_tiles, w_dtype, f_dtype, sign, max_ctas,
                         as_stream(stream));
}

int sdb_lora_patch_one(void* w_in, void* w_out, int64_t h1, int64_t h2, int64_t ldw,
                       const void* down, int64_t ldd, const void* up, int64_t ldu, int32_t rank,
                       float scale, float sign, int w_dtype, int f_dtype, void* stream) {
  sdb_lora_job j;
  std::memset(&j, 0, sizeof(j));
  j.w_in = w_in;
  j.w_out = w_out ? w_out : w_in;
  j.down = down;
  j.up = up;
  j.h1 = h1;
  j.h2 = h2;
  j.ldw = ldw;
  j.ldd = ldd;
  j.ldu = ldu;
  j.rank = rank;
  j.scale = scale;
  j.tile_begin = 0;
  if (int rc = check_job(j, 0)) return rc;
  return lora_patch_simt(nullptr, j, 1, simt_tiles(h1, h2), w_dtype, f_dtype, sign, 0,
                         as_stream(stream));
}

int sdb_lora_pack_bytes(int64_t h1, int64_t h2, int32_t rank, size_t* a_bytes, size_t* b_bytes) {
  if (h1 <= 0 || h2 <= 0 || rank < 1 || rank > 256 || !a_bytes || !b_bytes)
    return fail(SDB_EINVAL, "sdb_lora_pack_bytes: bad shape / rank (1..256)");
  tc_pack_bytes(h1, h2, rank, a_bytes, b_bytes);
  return SDB_OK;
}

int sdb_lora_pack(const void* down, int64_t ldd, const void* up, int64_t ldu, int64_t h1, int64_t h2,
                  int32_t rank, void* a_packed, void* b_packed, void* stream) {
  if (!down || !up || !a_packed || !b_packed) return fail(SDB_EINVAL, "sdb_lora_pack: NULL pointer");
  if (ldd < rank || ldu < h2) return fail(SDB_EINVAL, "sdb_lora_pack: leading dimension too small");
  return tc_pack(down, ldd, up, ldu, h1, h2, rank, a_packed, b_packed, as_stream(stream));
}

int sdb_lora_pack_multi(const sdb_lora_src* srcs_host, int n_src, int64_t h1, int64_t h2, void* a_packed,
                        void* b_packed, void* stream) {
  return tc_pack_multi(srcs_host, n_src, h1, h2, a_packed, b_packed, as_stream(stream));
}

int sdb_lora_pack_multi_layout(const sdb_lora_src* srcs_host, int n_src, int64_t h1, int64_t h2, size_t* a_bytes,
                               size_t* b_bytes, float* epi_scale, int32_t* lo_mask) {
  if (h1 <= 0 || h2 <= 0) return fail(SDB_EINVAL, "sdb_lora_pack_multi_layout: bad shape");
  return tc_pack_multi_layout(srcs_host, n_src, h1, h2, a_bytes, b_bytes, epi_scale, lo_mask);
}

int sdb_lora_tc_plan(const sdb_lora_tc_job* jobs_host, int n_jobs, void* blob_host, size_t blob_bytes,
                     size_t* needed, int* n_units, int* kb_max) {
  return tc_plan(jobs_host, n_jobs, blob_host, blob_bytes, needed, n_units, kb_max);
}

int sdb_lora_tc_set_mode(int mode) {
  return tc_set_mode(mode);
}

int sdb_lora_tc_patch(const void* blob_dev, int n_jobs, int n_units, int kb_max, int simt_rank, float sign,
                      int max_ctas, void* stream) {
  return tc_patch(blob_dev, n_jobs, n_units, kb_max, simt_rank, sign, max_ctas, as_stream(stream));
}

size_t sdb_groupnorm_workspace(int64_t n, int64_t hw, int64_t c, int64_t groups) {
  if (n <= 0 || hw <= 0 || c <= 0 || groups <= 0) return 0;
  return groupnorm_workspace(n, hw, c, groups);
}

int sdb_groupnorm_silu(const void* x, void* y, const float* gamma, const float* beta,
                       const float* add_nc, int64_t n, int64_t hw, int64_t c, int64_t groups,
                       float eps, int apply_silu, int dtype, void* workspace, void* stream) {
  return groupnorm_silu(x, y, gamma, beta, add_nc, n, hw, c, groups, eps, apply_silu, dtype, workspace,
                        as_stream(stream), 1);
}

int sdb_groupnorm_apply(const void* x, void* y, const float* gamma, const float* beta,
                        const float* add_nc, int64_t n, int64_t hw, int64_t c, int64_t groups,
                        float eps, int apply_silu, int dtype, void* workspace, void* stream) {
  return groupnorm_silu(x, y, gamma, beta, add_nc, n, hw, c, groups, eps, apply_silu, dtype, workspace,
                        as_stream(stream), 0);
}

int sdb_residual_inject_gn(void* out, const void* hidden, const void* skip,
                           const void* const* res_ptrs_host, const float* scales_host, int n_res,
                           int64_t n, int64_t hw, int64_t ch, int64_t cs, const float* hidden_bias,
                           const float* skip_bias, int64_t groups, void* gn_workspace, int dtype, void* stream) {
  return residual_inject_gn(out, hidden, skip, res_ptrs_host, scales_host, n_res, n, hw, ch, cs, hidden_bias,
                            skip_bias, groups, gn_workspace, dtype, as_stream(stream));
}

int sdb_residual_inject(void* out, const void* hidden, const void* skip,
                        const void* const* res_ptrs_host, const float* scales_host, int n_res,
                        int64_t pixels, int64_t ch, int64_t cs, int dtype, void* stream) {
  return residual_inject(out, hidden, skip, res_ptrs_host, scales_host, n_res, pixels, ch, cs, nullptr, nullptr,
                         dtype, as_stream(stream));
}

int sdb_residual_inject_bias(void* out, const void* hidden, const void* skip,
                             const void* const* res_ptrs_host, const float* scales_host, int n_res,
                             int64_t pixels, int64_t ch, int64_t cs, const float* hidden_bias,
                             const float* skip_bias, int dtype, void* stream) {
  return residual_inject(out, hidden, skip, res_ptrs_host, scales_host, n_res, pixels, ch, cs, hidden_bias,
                         skip_bias, dtype, as_stream(stream));
}

int64_t sdb_batched_copy_chunk_vectors(void) { return batched_copy_chunk_vectors(); }

int sdb_batched_copy(const void* const* src_dev, void* const* dst_dev, const int64_t* nvec_dev,
                     const int64_t* chunk_prefix_dev, int n, int64_t total_chunks, void* stream) {
  if (n < 0 || (n > 0 && (!src_dev || !dst_dev || !nvec_dev || !chunk_prefix_dev)))
    return fail(SDB_EINVAL, "sdb_batched_copy: NULL table");
  return batched_copy(src_dev, dst_dev, nvec_dev, chunk_prefix_dev, n, total_chunks, as_stream(stream));
}

int sdb_upsample2x(const void* x, void* y, int64_t n, int64_t h, int64_t w, int64_t c, int elem_bytes,
                   void* stream) {
  return upsample2x(x, y, n, h, w, c, elem_bytes, as_stream(stream));
}

int sdb_geglu(const void* proj, void* out, int64_t rows, int64_t f, int dtype, void* stream) {
  return geglu(proj, out, rows, f, dtype, as_stream(stream));
}

int sdb_ff_geglu(const void* x, const void* w, const float* bias, void* out, int64_t m, int64_t k, int64_t f,
                 void* stream) {
  return ff_geglu(x, w, bias, out, m, k, f, as_stream(stream));
}

int sdb_add_layernorm(void* x, const void* d, void* y, const void* gamma, const void* beta, int64_t rows,
                      int64_t c, float eps, int dtype, void* stream) {
  return add_layernorm(x, d, y, gamma, beta, rows, c, eps, dtype, as_stream(stream));
}

int sdb_cross_attention(const void* q, int64_t ldq, const void* kv, int64_t ldkv, int64_t voff, void* o,
                        int64_t ldo, int n, int lq, int lk, int heads, int head_dim, float scale, int dtype,
                        void* stream) {
  return cross_attention(q, ldq, kv, ldkv, voff, o, ldo, n, lq, lk, heads, head_dim, scale, dtype,
                         as_stream(stream));
}

int sdb_cross_attention_set_mode(int tcgen05) { return cross_attention_set_mode(tcgen05); }

int sdb_self_attention(const void* qkv, int64_t ldqkv, void* o, int64_t ldo, int n, int seq_len, int heads,
                       int head_dim, float scale, int dtype, void* stream) {
  return self_attention(qkv, ldqkv, o, ldo, n, seq_len, heads, head_dim, scale, dtype, as_stream(stream));
}

int sdb_stream_wait_value32(void* stream, void* addr, uint32_t value) {
  return stream_wait_value32(as_stream(stream), addr, value);
}

int sdb_stream_write_value32(void* stream, void* addr, uint32_t value) {
  return stream_write_value32(as_stream(stream), addr, value);
}

int sdb_memcpy_async(void* dst, const void* src, size_t bytes, void* stream) {
  return memcpy_async(dst, src, bytes, as_stream(stream));
}

int sdb_cfg_ddim_step(const void* eps, int eps_dtype, const float* x, float* x_out, void* unet_in,
                      int in_dtype, int64_t latent_elems, const float* coef, int* step_dev,
                      void* stream) {
  return cfg_ddim_step(eps, eps_dtype, x, x_out, unet_in, in_dtype, latent_elems, coef, step_dev,
                       as_stream(stream));
}

void sdb_groupnorm_set_mode(int mode) { g_gn_cluster_mode = mode; }

int sdb_set_pdl(int on) {
  const int prev = g_pdl;
  g_pdl = on != 0;
  return prev;
}

int sdb_groupnorm_launches(int64_t n, int64_t hw, int64_t c, int64_t groups, int dtype) {
  return gn_launches(n, hw, c, groups, dtype);
}

int sdb_groupnorm_stream_plan(int64_t n, int64_t hw, int64_t c, int64_t groups, int* out7) {
  return gn_stream_plan(n, hw, c, groups, out7);
}

int sdb_groupnorm_resident_plan(int64_t n, int64_t hw, int64_t c, int64_t groups, int* out4) {
  return gn_resident_plan(n, hw, c, groups, out4);
}

int sdb_conv_out(const void* x, const void* w, const float* bias, float* out, int64_t n, int64_t h,
                 int64_t width, int64_t c, int64_t cout, int dtype, void* stream) {
  return conv_out(x, w, bias, out, n, h, width, c, cout, dtype, as_stream(stream));
}

}  // extern "C"
