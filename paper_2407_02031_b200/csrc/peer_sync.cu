// peer_sync.cu — GPU-side cross-process / cross-GPU step handshakes for the
// ControlNet-as-a-service transport (caas.CaaSPeerProtocol).
//
// The base and its ControlNet services exchange data through each other's
// memory (CUDA IPC mappings, NVLink peer copies) and order it with 32-bit
// sequence flags written and awaited by the GPUs themselves — stream memory
// operations (cuStreamWriteValue32 / cuStreamWaitValue32), no NCCL call and
// no host round trip per step.  The writer's write is preceded by a
// system-scope fence (CU_STREAM_WRITE_VALUE_DEFAULT), so every peer store or
// copy the stream issued before it is visible once the waiter sees the value.
// This replaces the per-step message/transfer steps the reference models as
// comm_ms (addonsim/model.py:151-158; orchestrator.py:621-660).
#include <cuda.h>

#include "common.cuh"

namespace sdb {
namespace {

typedef CUresult (*StreamValue32Fn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

StreamValue32Fn entry(const char* name) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) == cudaSuccess && q == cudaDriverEntryPointSuccess)
    return reinterpret_cast<StreamValue32Fn>(p);
  cudaGetLastError();
  return nullptr;
}

}  // namespace

int stream_wait_value32(cudaStream_t st, void* addr, uint32_t value) {
  static StreamValue32Fn fn = entry("cuStreamWaitValue32");
  if (!fn) return fail(SDB_ECUDA, "cuStreamWaitValue32 unavailable");
  if (!addr || (reinterpret_cast<uintptr_t>(addr) & 3)) return fail(SDB_EINVAL, "stream_wait_value32: bad address");
  const CUresult r = fn(reinterpret_cast<CUstream>(st), reinterpret_cast<CUdeviceptr>(addr), value,
                        CU_STREAM_WAIT_VALUE_GEQ);
  if (r != CUDA_SUCCESS) return fail(SDB_ECUDA, "cuStreamWaitValue32 failed (" + std::to_string((int)r) + ")");
  return SDB_OK;
}

int stream_write_value32(cudaStream_t st, void* addr, uint32_t value) {
  static StreamValue32Fn fn = entry("cuStreamWriteValue32");
  if (!fn) return fail(SDB_ECUDA, "cuStreamWriteValue32 unavailable");
  if (!addr || (reinterpret_cast<uintptr_t>(addr) & 3)) return fail(SDB_EINVAL, "stream_write_value32: bad address");
  const CUresult r = fn(reinterpret_cast<CUstream>(st), reinterpret_cast<CUdeviceptr>(addr), value,
                        CU_STREAM_WRITE_VALUE_DEFAULT);
  if (r != CUDA_SUCCESS) return fail(SDB_ECUDA, "cuStreamWriteValue32 failed (" + std::to_string((int)r) + ")");
  return SDB_OK;
}

int memcpy_async(void* dst, const void* src, size_t bytes, cudaStream_t st) {
  if (bytes == 0) return SDB_OK;
  if (!dst || !src) return fail(SDB_EINVAL, "memcpy_async: NULL pointer");
  // UVA: local, peer-mapped (NVLink) and IPC-mapped pointers alike
  const cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, st);
  if (e != cudaSuccess) return fail(SDB_ECUDA, std::string("memcpy_async: ") + cudaGetErrorString(e));
  return SDB_OK;
}

}  // namespace sdb
