// cfg_step.cu — K4: classifier-free guidance combine fused with the DDIM
// (eta = 0) update and the CFG re-batching of the next UNet input.
//
// Not present in the reference at all (no guidance / scheduler
// arithmetic anywhere in addonsim).  Conventions follow the usual diffusers
// pipeline: eps = eps_u + g (eps_c - eps_u) over a [uncond; cond] batch of 2,
// DDIM step with alphas_cumprod a_t -> a_prev.
//
// The step index lives on the device (step_dev[0]); the last CTA to finish
// advances it (threadfence + done counter in step_dev[1]), so one denoising
// step — UNet, ControlNets, this kernel — replays as a CUDA graph with no
// host work between steps.
#include "common.cuh"

namespace sdb {
namespace {

template <typename TE, typename TI>
__global__ void __launch_bounds__(256)
cfg_ddim_kernel(const TE* __restrict__ eps, const float* x, float* x_out,   // x_out may alias x (in place)
                TI* __restrict__ unet_in, int64_t L, const float* __restrict__ coef,
                int* __restrict__ step_dev) {
  pdl_wait();
  const int step = *reinterpret_cast<volatile int*>(step_dev);
  const float a_t = coef[step * 4 + 0];
  const float a_prev = coef[step * 4 + 1];
  const float g = coef[step * 4 + 2];
  const float sa = sqrtf(a_t), s1a = sqrtf(1.f - a_t);
  const float sp = sqrtf(a_prev), s1p = sqrtf(1.f - a_prev);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < L;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float eu = to_f32<TE>(eps[i]);
    const float ec = to_f32<TE>(eps[L + i]);
    const float e = fmaf(g, ec - eu, eu);
    const float xi = x[i];
    const float x0 = (xi - s1a * e) / sa;
    const float xp = fmaf(sp, x0, s1p * e);
    x_out[i] = xp;
    if (unet_in != nullptr) {
      const TI v = from_f32<TI>(xp);
      unet_in[i] = v;
      unet_in[L + i] = v;
    }
  }
  // grid-wide completion: the last CTA advances the device step counter
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const int done = atomicAdd(step_dev + 1, 1);
    if (done == (int)gridDim.x - 1) {
      step_dev[1] = 0;
      step_dev[0] = step + 1;
      __threadfence();
    }
  }
}

template <typename TE, typename TI>
int run_cfg(const void* eps, const float* x, float* x_out, void* unet_in, int64_t L,
            const float* coef, int* step_dev, cudaStream_t st) {
  int64_t grid = (L + 255) / 256;
  if (grid > kNumSMs * 4) grid = kNumSMs * 4;
  if (grid < 1) grid = 1;
  launch_k(cfg_ddim_kernel<TE, TI>, (unsigned)grid, 256, 0, st, static_cast<const TE*>(eps), x, x_out,
                                                          static_cast<TI*>(unet_in), L, coef, step_dev);
  return check_launch("cfg_ddim_kernel");
}

}  // namespace

int cfg_ddim_step(const void* eps, int eps_dtype, const float* x, float* x_out, void* unet_in,
                  int in_dtype, int64_t L, const float* coef, int* step_dev, cudaStream_t st) {
  if (L <= 0) return fail(SDB_EINVAL, "cfg_ddim_step: empty latent");
  if (!eps || !x || !x_out || !coef || !step_dev) return fail(SDB_EINVAL, "cfg_ddim_step: NULL pointer");
#define SDB_CFG_CASE(E, ET, I, IT) \
  if (eps_dtype == E && in_dtype == I) return run_cfg<ET, IT>(eps, x, x_out, unet_in, L, coef, step_dev, st);
  SDB_CFG_CASE(SDB_BF16, __nv_bfloat16, SDB_BF16, __nv_bfloat16)
  SDB_CFG_CASE(SDB_F32, float, SDB_F32, float)
  SDB_CFG_CASE(SDB_F16, __half, SDB_F16, __half)
  SDB_CFG_CASE(SDB_BF16, __nv_bfloat16, SDB_F32, float)
  SDB_CFG_CASE(SDB_F32, float, SDB_BF16, __nv_bfloat16)
#undef SDB_CFG_CASE
  return fail(SDB_EUNSUP, "cfg_ddim_step: unsupported dtype combination");
}

}  // namespace sdb
