"""Which attention kernel is fastest for the SDXL shapes (development aid)."""

import torch
import torch.nn.functional as F
from torch.nn.attention import SDPBackend, sdpa_kernel


def t(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps * 1000


def main():
    dev = "cuda"
    for name, (h, L, Lk) in {"self64": (10, 4096, 4096), "self32": (20, 1024, 1024),
                             "cross64": (10, 4096, 77), "cross32": (20, 1024, 77)}.items():
        q = torch.randn(2, L, h, 64, device=dev, dtype=torch.bfloat16).transpose(1, 2)
        k = torch.randn(2, Lk, h, 64, device=dev, dtype=torch.bfloat16).transpose(1, 2)
        v = torch.randn(2, Lk, h, 64, device=dev, dtype=torch.bfloat16).transpose(1, 2)
        res = {}
        for bname, be in [("default", None), ("cudnn", SDPBackend.CUDNN_ATTENTION),
                          ("flash", SDPBackend.FLASH_ATTENTION), ("efficient", SDPBackend.EFFICIENT_ATTENTION)]:
            try:
                if be is None:
                    res[bname] = t(lambda: F.scaled_dot_product_attention(q, k, v))
                else:
                    with sdpa_kernel([be]):
                        res[bname] = t(lambda: F.scaled_dot_product_attention(q, k, v))
            except Exception as e:  # noqa: BLE001
                res[bname] = repr(e)[:60]
        try:
            from flash_attn import flash_attn_func
            qq, kk, vv = (x.transpose(1, 2) for x in (q, k, v))
            res["flash_attn_lib"] = t(lambda: flash_attn_func(qq, kk, vv))
        except Exception as e:  # noqa: BLE001
            res["flash_attn_lib"] = repr(e)[:60]
        if Lk == 77:
            kp = torch.zeros(2, h, 128, 64, device=dev, dtype=torch.bfloat16)
            vp = torch.zeros_like(kp)
            kp[:, :, :77] = k
            vp[:, :, :77] = v
            mask = torch.zeros(1, 1, 1, 128, device=dev, dtype=torch.bfloat16)
            mask[..., 77:] = float("-inf")
            res["padded128_mask"] = t(lambda: F.scaled_dot_product_attention(q, kp, vp, attn_mask=mask))
        print(name, {k: (round(v, 1) if isinstance(v, float) else v) for k, v in res.items()}, flush=True)


if __name__ == "__main__":
    main()
