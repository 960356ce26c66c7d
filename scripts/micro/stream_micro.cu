// stream_micro.cu — how fast can a 21 MB NHWC map be read (stats-like) or
// read+written (apply-like) on this B200, as a function of grid / block /
// loads in flight?  Each config: 24 launches captured in one CUDA graph, each
// on its own copy of the input (8 copies = 168 MB > L2), timed as replays.
// Development aid for K2; not part of the library.
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__device__ __forceinline__ uint4 ldg_hint(const uint4* p, uint64_t pol) {
  uint4 r;
  asm volatile("ld.global.nc.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ uint64_t pol_first() {
  uint64_t p; asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p)); return p;
}
__device__ __forceinline__ uint64_t pol_last() {
  uint64_t p; asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p)); return p;
}
__device__ __forceinline__ float sum8(uint4 v) {
  const uint32_t* u = &v.x; float s = 0.f;
#pragma unroll
  for (int i = 0; i < 4; ++i) s += __uint_as_float(u[i] << 16) + __uint_as_float(u[i] & 0xffff0000u);
  return s;
}

template <int U, int HINT>
__global__ void read_kernel(const uint4* __restrict__ x, long nvec, float* out) {
  const uint64_t pol = HINT == 1 ? pol_last() : pol_first();
  float s = 0.f;
  const long stride = (long)gridDim.x * blockDim.x;
  long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  // contiguous per-CTA span variant would differ; grid-stride keeps all SMs busy
  for (; i + (U - 1) * stride < nvec; i += U * stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = HINT ? ldg_hint(x + i + u * stride, pol) : x[i + u * stride];
#pragma unroll
    for (int u = 0; u < U; ++u) s += sum8(v[u]);
  }
  for (; i < nvec; i += stride) s += sum8(x[i]);
  if (s == 12345.f) out[0] = s;   // keep the loads
}

// contiguous span per CTA (like K2's chunking)
template <int U>
__global__ void read_span_kernel(const uint4* __restrict__ x, long nvec, float* out) {
  const long per = (nvec + gridDim.x - 1) / gridDim.x;
  const long b = (long)blockIdx.x * per, e = min(nvec, b + per);
  const uint64_t pol = pol_last();
  float s = 0.f;
  long i = b + threadIdx.x;
  for (; i + (U - 1) * (long)blockDim.x < e; i += U * (long)blockDim.x) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ldg_hint(x + i + u * blockDim.x, pol);
#pragma unroll
    for (int u = 0; u < U; ++u) s += sum8(v[u]);
  }
  for (; i < e; i += blockDim.x) s += sum8(x[i]);
  if (s == 12345.f) out[0] = s;
}

template <int U>
__global__ void copy_kernel(const uint4* __restrict__ x, uint4* __restrict__ y, long nvec) {
  const uint64_t pol = pol_first();
  const long stride = (long)gridDim.x * blockDim.x;
  long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < nvec; i += U * stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ldg_hint(x + i + u * stride, pol);
#pragma unroll
    for (int u = 0; u < U; ++u) { v[u].x ^= 1u; y[i + u * stride] = v[u]; }
  }
  for (; i < nvec; i += stride) y[i] = x[i];
}

__global__ void empty_kernel(float* out) { if (threadIdx.x == 12345) out[0] = 1.f; }

template <typename F>
float time_graph(F launch, int reps = 24) {
  cudaStream_t s; cudaStreamCreate(&s);
  for (int i = 0; i < 3; ++i) launch(s, i);
  cudaStreamSynchronize(s);
  cudaGraph_t g; cudaGraphExec_t ge;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
  for (int i = 0; i < reps; ++i) launch(s, i);
  cudaStreamEndCapture(s, &g);
  cudaGraphInstantiate(&ge, g, 0);
  cudaGraphLaunch(ge, s);
  cudaStreamSynchronize(s);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a, s);
  for (int k = 0; k < 5; ++k) cudaGraphLaunch(ge, s);
  cudaEventRecord(b, s);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  cudaGraphExecDestroy(ge); cudaGraphDestroy(g); cudaStreamDestroy(s);
  return ms * 1000.f / (5 * reps);
}

int main() {
  const long bytes = 2L * 320 * 128 * 128 * 2;   // 21 MB
  const long nvec = bytes / 16;
  const int ncopy = 8;
  std::vector<uint4*> xs(ncopy), ys(ncopy);
  for (int i = 0; i < ncopy; ++i) {
    cudaMalloc(&xs[i], bytes); cudaMalloc(&ys[i], bytes);
    cudaMemset(xs[i], 1, bytes);
  }
  float* out; cudaMalloc(&out, 4);
  printf("map %.1f MB; peak-time read %.2f us, read+write %.2f us at 6548.8 GB/s\n", bytes / 1e6,
         bytes / 6548.8e3, 2 * bytes / 6548.8e3);
  printf("empty kernel in graph: %.2f us\n", time_graph([&](cudaStream_t s, int i) {
    empty_kernel<<<148, 256, 0, s>>>(out); }));
  int grids[] = {148, 296, 592, 1184};
  int blocks[] = {256, 512, 1024};
  for (int gi : grids) for (int bl : blocks) {
    if ((long)gi * bl > 148L * 2048) continue;
    float r2 = time_graph([&](cudaStream_t s, int i) { read_kernel<4, 1><<<gi, bl, 0, s>>>(xs[i % ncopy], nvec, out); });
    float r8 = time_graph([&](cudaStream_t s, int i) { read_kernel<8, 1><<<gi, bl, 0, s>>>(xs[i % ncopy], nvec, out); });
    float rp = time_graph([&](cudaStream_t s, int i) { read_kernel<4, 0><<<gi, bl, 0, s>>>(xs[i % ncopy], nvec, out); });
    float rs = time_graph([&](cudaStream_t s, int i) { read_span_kernel<4><<<gi, bl, 0, s>>>(xs[i % ncopy], nvec, out); });
    float c4 = time_graph([&](cudaStream_t s, int i) { copy_kernel<4><<<gi, bl, 0, s>>>(xs[i % ncopy], ys[i % ncopy], nvec); });
    float c8 = time_graph([&](cudaStream_t s, int i) { copy_kernel<8><<<gi, bl, 0, s>>>(xs[i % ncopy], ys[i % ncopy], nvec); });
    printf("grid %5d block %4d | read U4 hint %.2f us (%.0f GB/s) U8 %.2f  plain %.2f  span %.2f | copy U4 %.2f us (%.0f GB/s) U8 %.2f\n",
           gi, bl, r2, bytes / r2 / 1e3, r8, rp, rs, c4, 2 * bytes / c4 / 1e3, c8);
  }
  // read then copy (stats + apply pattern; the apply re-reads the same buffer)
  for (int gi : {296, 592}) {
    float rc = time_graph([&](cudaStream_t s, int i) {
      read_kernel<4, 1><<<148, 1024, 0, s>>>(xs[i % ncopy], nvec, out);
      copy_kernel<4><<<gi, 256, 0, s>>>(xs[i % ncopy], ys[i % ncopy], nvec); });
    printf("read(148x1024) + copy(%d x 256) back to back: %.2f us (%.0f GB/s of 2x map)\n", gi, rc, 2 * bytes / rc / 1e3);
  }
  return 0;
}
