// lora_patch_tc.cu — K1 tensor-core path (tcgen05 + TMEM), placeholder until
// the kernel lands; sdb_lora_plan never selects it while tc_supported() is false.
#include "common.cuh"

namespace sdb {

int64_t tc_tiles(int64_t h1, int64_t h2) { return ((h1 + 127) / 128) * ((h2 + 255) / 256); }

bool tc_supported(int, int, int) { return false; }

int lora_patch_tc(const sdb_lora_job*, int, int64_t, float, int, cudaStream_t) {
  return fail(SDB_EUNSUP, "tcgen05 LoRA path not built");
}

}  // namespace sdb
