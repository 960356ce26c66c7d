"""paper_2407_02031_b200 — B200-native SwiftDiffusion add-on hot path.

Host side (Python/PyTorch) of the per-step denoising loop with ControlNet
residual injection and LoRA patch/unpatch; every kernel on the path is
hand-written sm_100a CUDA in libsdb.so behind the C-ABI of include/sdb_api.h.

Modules
  lora       drop-in for addonsim.lora (merge_in_place, unmerge_in_place, ...)
  schedule   drop-in for the step-loop semantics (plan_lora_patch, LatencyProfile, ...)
  ops        torch-tensor wrappers of the C-ABI kernels K1-K4
  patcher    batched whole-UNet LoRA patch sets (shadow weights, side stream)
  unet       SD1.5 / SDXL / toy-shaped UNet + ControlNet (NHWC, bf16)
  pipeline   CFG denoising loop with ControlNets and the async LoRA patch
  caas       ControlNet-as-a-service over torch.distributed (one rank per GPU)
"""

__version__ = "0.1.0"
