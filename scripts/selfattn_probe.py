"""Self-attention candidates at the SDXL shapes, timed as CUDA-graph replays
(no host overhead).  Development aid: library options vs torch's cuDNN SDPA."""
import sys
import time
import traceback

import torch
import torch.nn.functional as F


def graph_time(fn, reps=20):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        g.replay()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / (5 * reps) * 1000


def main():
    import flashinfer
    for name, (n, L, h) in {"self64": (2, 4096, 10), "self32": (2, 1024, 20)}.items():
        d = 64
        qkv = torch.randn(n, L, 3, h, d, device="cuda", dtype=torch.bfloat16)
        q, k, v = (qkv[:, :, i].transpose(1, 2) for i in range(3))
        res = {}
        res["torch_sdpa"] = graph_time(lambda: F.scaled_dot_product_attention(q, k, v))
        flops = 4 * n * h * L * L * d
        qf = qkv[:, :, 0].reshape(n * L, h, d).contiguous()
        kf = qkv[:, :, 1].reshape(n * L, h, d).contiguous()
        vf = qkv[:, :, 2].reshape(n * L, h, d).contiguous()
        indptr = torch.arange(0, (n + 1) * L, L, device="cuda", dtype=torch.int32)
        ref = F.scaled_dot_product_attention(q.float(), k.float(), v.float()).transpose(1, 2).reshape(n * L, h, d)
        for be in ["cutlass", "fa2", "cudnn", "trtllm-gen", "fa3"]:
            t0 = time.time()
            try:
                ws = torch.zeros(256 << 20, dtype=torch.uint8, device="cuda")
                w = flashinfer.BatchPrefillWithRaggedKVCacheWrapper(ws, "NHD", backend=be)
                w.plan(indptr, indptr, h, h, d, causal=False, q_data_type=torch.bfloat16)
                o = w.run(qf, kf, vf)
                err = (o.float() - ref).abs().max().item()
                res[be] = (round(graph_time(lambda: w.run(qf, kf, vf)), 2), f"err {err:.3g}", f"setup {time.time()-t0:.0f}s")
            except Exception as e:  # noqa: BLE001
                res[be] = repr(e)[:120]
            print(name, be, res[be], flush=True)
        print(name, "torch_sdpa", round(res["torch_sdpa"], 2), "us;", "TFLOP/s", round(flops / res["torch_sdpa"] / 1e6, 1), flush=True)




def k8():
    import sys as _s
    from pathlib import Path
    _s.path.insert(0, str(Path(__file__).resolve().parent.parent))
    from paper_2407_02031_b200 import ops
    for name, (n, L, h) in {"self64": (2, 4096, 10), "self32": (2, 1024, 20)}.items():
        qkv = torch.randn(n, L, 3 * h * 64, device="cuda", dtype=torch.bfloat16)
        q, k, v = (t.reshape(n, L, h, 64).transpose(1, 2) for t in qkv.split(h * 64, dim=-1))
        t_k8 = graph_time(lambda: ops.self_attention(qkv, h))
        t_sdpa = graph_time(lambda: F.scaled_dot_product_attention(q, k, v))
        flops = 4 * n * h * L * L * 64
        print(name, "K8", round(t_k8, 2), "us", round(flops / t_k8 / 1e6, 1), "TF/s | sdpa", round(t_sdpa, 2), "us",
              round(flops / t_sdpa / 1e6, 1), "TF/s", flush=True)


if __name__ == "__main__":
    k8() if len(sys.argv) > 1 and sys.argv[1] == "k8" else main()
