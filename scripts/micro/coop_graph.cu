// coop_graph.cu — can a cooperative (grid-synchronising) kernel be captured in
// a CUDA graph and replayed, and what does one grid.sync cost?  Dev aid.
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void coop_kernel(int* counter, int* out, int rounds) {
  cg::grid_group g = cg::this_grid();
  for (int r = 0; r < rounds; ++r) {
    if (threadIdx.x == 0) atomicAdd(counter, 1);
    g.sync();
    if (blockIdx.x == 0 && threadIdx.x == 0) out[r] = *counter;
    g.sync();
  }
}

int main() {
  int *counter, *out;
  cudaMalloc(&counter, 4);
  cudaMalloc(&out, 64 * 4);
  cudaMemset(counter, 0, 4);
  cudaStream_t s;
  cudaStreamCreate(&s);
  int rounds = 1;
  void* args[] = {&counter, &out, &rounds};
  dim3 grid(148), block(1024);
  cudaError_t e = cudaLaunchCooperativeKernel((void*)coop_kernel, grid, block, args, 0, s);
  printf("eager cooperative launch: %s\n", cudaGetErrorString(e));
  cudaStreamSynchronize(s);
  cudaGraph_t gph;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
  for (int i = 0; i < 20; ++i) e = cudaLaunchCooperativeKernel((void*)coop_kernel, grid, block, args, 0, s);
  cudaError_t e2 = cudaStreamEndCapture(s, &gph);
  printf("capture: launch %s, end %s\n", cudaGetErrorString(e), cudaGetErrorString(e2));
  e = cudaGraphInstantiate(&ge, gph, 0);
  printf("instantiate: %s\n", cudaGetErrorString(e));
  cudaGraphLaunch(ge, s);
  e = cudaStreamSynchronize(s);
  printf("replay: %s\n", cudaGetErrorString(e));
  int h;
  cudaMemcpy(&h, counter, 4, cudaMemcpyDeviceToHost);
  printf("counter %d (expect %d)\n", h, 148 * 21);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int rr : {1, 8}) {
    rounds = rr;
    cudaGraph_t g2;
    cudaGraphExec_t ge2;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < 20; ++i) cudaLaunchCooperativeKernel((void*)coop_kernel, grid, block, args, 0, s);
    cudaStreamEndCapture(s, &g2);
    cudaGraphInstantiate(&ge2, g2, 0);
    cudaGraphLaunch(ge2, s);
    cudaEventRecord(a, s);
    for (int k = 0; k < 5; ++k) cudaGraphLaunch(ge2, s);
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("rounds %d: %.2f us per launch (2 grid syncs per round)\n", rr, ms * 1000 / 100);
  }
  return 0;
}
