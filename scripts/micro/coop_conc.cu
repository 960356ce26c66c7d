// coop_conc.cu — is a grid barrier safe when several one-CTA-per-SM grids run
// concurrently on different streams (as K2's resident form would inside the
// CaaS loopback engine: encoder graph || ControlNet graphs)?  Dev aid.
//
// Each grid: 148 CTAs x 1024 threads with 150 KB dynamic smem (one per SM),
// thread 0 arrives on a per-stream counter and spins on the generation word
// with a 5 ms timeout (so a deadlock shows up as a timeout count, not a hang).
// Modes: plain launches, cooperative-attribute launches, cooperative launches
// captured in one graph with 3 parallel branches, cooperative + PDL.
#include <cuda_runtime.h>
#include <cstdio>

struct Bar {
  unsigned int arrivals, gen, timeouts, pad;
};

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void __launch_bounds__(1024, 1) spin_barrier(Bar* b, int work) {
  extern __shared__ unsigned char smem[];
  asm volatile("griddepcontrol.wait;" ::: "memory");
  // a little work so the grids overlap in time
  float acc = threadIdx.x;
  for (int i = 0; i < work; ++i) acc = acc * 1.0001f + 1.f;
  smem[threadIdx.x] = (unsigned char)acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int g0;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(g0) : "l"(&b->gen));
    __threadfence();
    if (atomicAdd(&b->arrivals, 1u) == gridDim.x - 1) {
      b->arrivals = 0u;
      __threadfence();
      atomicAdd(&b->gen, 1u);
    } else {
      const unsigned long long t0 = gtime();
      while (true) {
        unsigned int g;
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(&b->gen));
        if (g != g0) break;
        if (gtime() - t0 > 5000000ull) {
          atomicAdd(&b->timeouts, 1u);
          break;
        }
      }
    }
  }
  __syncthreads();
  if (smem[threadIdx.x] == 255 && work < 0) b->pad = 1;
}

static cudaError_t launch(Bar* b, cudaStream_t s, bool coop, bool pdl, int work) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(148);
  cfg.blockDim = dim3(1024);
  cfg.dynamicSmemBytes = 150 * 1024;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  int na = 0;
  if (coop) {
    at[na].id = cudaLaunchAttributeCooperative;
    at[na].val.cooperative = 1;
    ++na;
  }
  if (pdl) {
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, spin_barrier, b, work);
}

int main() {
  cudaFuncSetAttribute(spin_barrier, cudaFuncAttributeMaxDynamicSharedMemorySize, 150 * 1024);
  const int NS = 3, ITER = 200;
  Bar* bars;
  cudaMalloc(&bars, NS * sizeof(Bar));
  cudaStream_t st[NS];
  for (int i = 0; i < NS; ++i) cudaStreamCreateWithFlags(&st[i], cudaStreamNonBlocking);
  Bar h[NS];
  const char* names[] = {"plain", "cooperative", "cooperative+pdl"};
  for (int mode = 0; mode < 3; ++mode) {
    cudaMemset(bars, 0, NS * sizeof(Bar));
    cudaDeviceSynchronize();
    cudaEvent_t a, e;
    cudaEventCreate(&a);
    cudaEventCreate(&e);
    cudaEventRecord(a, st[0]);
    cudaError_t err = cudaSuccess;
    for (int it = 0; it < ITER; ++it)
      for (int s = 0; s < NS; ++s) {
        cudaError_t r = launch(bars + s, st[s], mode >= 1, mode == 2, 2000);
        if (r != cudaSuccess) err = r;
      }
    for (int s = 1; s < NS; ++s) {
      cudaEvent_t x;
      cudaEventCreate(&x);
      cudaEventRecord(x, st[s]);
      cudaStreamWaitEvent(st[0], x, 0);
    }
    cudaEventRecord(e, st[0]);
    cudaError_t se = cudaDeviceSynchronize();
    float ms = 0;
    cudaEventElapsedTime(&ms, a, e);
    cudaMemcpy(h, bars, sizeof(h), cudaMemcpyDeviceToHost);
    printf("%-18s launch %s sync %s: timeouts %u %u %u, gens %u %u %u, %.1f us per launch\n", names[mode],
           cudaGetErrorString(err), cudaGetErrorString(se), h[0].timeouts, h[1].timeouts, h[2].timeouts, h[0].gen,
           h[1].gen, h[2].gen, ms * 1000.f / (ITER * NS));
  }
  // cooperative launches captured into one graph with NS parallel branches
  {
    cudaMemset(bars, 0, NS * sizeof(Bar));
    cudaDeviceSynchronize();
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStream_t cs = st[0];
    cudaStreamBeginCapture(cs, cudaStreamCaptureModeGlobal);
    cudaEvent_t fork;
    cudaEventCreate(&fork);
    cudaEventRecord(fork, cs);
    for (int s = 1; s < NS; ++s) cudaStreamWaitEvent(st[s], fork, 0);
    cudaError_t err = cudaSuccess;
    for (int it = 0; it < 20; ++it)
      for (int s = 0; s < NS; ++s) {
        cudaError_t r = launch(bars + s, st[s], true, false, 2000);
        if (r != cudaSuccess) err = r;
      }
    for (int s = 1; s < NS; ++s) {
      cudaEvent_t x;
      cudaEventCreate(&x);
      cudaEventRecord(x, st[s]);
      cudaStreamWaitEvent(cs, x, 0);
    }
    cudaError_t ee = cudaStreamEndCapture(cs, &g);
    cudaError_t ie = cudaGraphInstantiate(&ge, g, 0);
    for (int r = 0; r < 10; ++r) cudaGraphLaunch(ge, cs);
    cudaError_t se = cudaDeviceSynchronize();
    cudaMemcpy(h, bars, sizeof(h), cudaMemcpyDeviceToHost);
    printf("graph 3 branches   capture %s/%s instantiate %s sync %s: timeouts %u %u %u, gens %u %u %u\n",
           cudaGetErrorString(err), cudaGetErrorString(ee), cudaGetErrorString(ie), cudaGetErrorString(se),
           h[0].timeouts, h[1].timeouts, h[2].timeouts, h[0].gen, h[1].gen, h[2].gen);
  }
  return 0;
}
