"""SDXL linear shapes under torch's two BLAS front ends (dev aid): the default
(cuBLAS) vs preferred_blas_library('cublaslt'); CUDA-graph replays."""
import sys
import torch
import torch.nn.functional as F

sys.path.insert(0, ".")
from scripts.gemm_tune_probe import SHAPES, gtime  # noqa: E402

print("default:", torch.backends.cuda.preferred_blas_library())
for lib in ("cublas", "cublaslt"):
    torch.backends.cuda.preferred_blas_library(lib)
    line = lib
    for m, k, n, bias in SHAPES:
        x = torch.randn(m, k, device="cuda", dtype=torch.bfloat16)
        w = torch.randn(n, k, device="cuda", dtype=torch.bfloat16) * 0.02
        b = torch.zeros(n, device="cuda", dtype=torch.bfloat16) if bias else None
        us = gtime(lambda: F.linear(x, w, b))
        line += f" | {m}x{k}x{n}{'b' if bias else ''} {us:.1f}"
    print(line, flush=True)
