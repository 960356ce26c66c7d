"""cuDNN frontend SDPA execution plans at the SDXL self-attention shapes
(dev aid): every plan the heuristics offer, timed, vs torch's SDPA (which
takes cuDNN's first heuristic pick).  Layout as the UNet produces it: q, k, v
are column slices of the fused to_qkv output [N, L, 3C]."""
import torch
import torch.nn.functional as F
import cudnn


def timeit(fn, reps=20):
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


handle = cudnn.create_handle()
cudnn.set_stream(handle=handle, stream=torch.cuda.current_stream().cuda_stream)
for n, l, h in [(2, 4096, 10), (2, 1024, 20)]:
    c = h * 64
    qkv = torch.randn(n, l, 3 * c, device="cuda", dtype=torch.bfloat16)
    q, k, v = (t.view(n, l, h, 64).transpose(1, 2) for t in qkv.split(c, dim=-1))
    o_t = torch.empty(n, l, c, device="cuda", dtype=torch.bfloat16)
    o = o_t.view(n, l, h, 64).transpose(1, 2)
    t_torch = timeit(lambda: F.scaled_dot_product_attention(q, k, v))
    g = cudnn.pygraph(io_data_type=cudnn.data_type.BFLOAT16, intermediate_data_type=cudnn.data_type.FLOAT,
                      compute_data_type=cudnn.data_type.FLOAT, handle=handle)
    Q = g.tensor_like(q)
    K = g.tensor_like(k)
    V = g.tensor_like(v)
    O, _ = g.sdpa(name="sdpa", q=Q, k=K, v=V, is_inference=True, attn_scale=64 ** -0.5)
    O.set_output(True).set_dim(list(o.shape)).set_stride(list(o.stride())).set_data_type(cudnn.data_type.BFLOAT16)
    g.validate()
    g.build_operation_graph()
    g.create_execution_plans([cudnn.heur_mode.A, cudnn.heur_mode.B, cudnn.heur_mode.FALLBACK])
    g.check_support()
    g.build_plans(cudnn.build_plan_policy.ALL)
    cnt = g.get_execution_plan_count()
    ws = torch.empty(max(g.get_workspace_size(), 1), device="cuda", dtype=torch.uint8)
    ref = F.scaled_dot_product_attention(q, k, v)
    print(f"[{n},{l},{h} heads] torch SDPA {t_torch:.1f} us; {cnt} cuDNN plans", flush=True)
    for i in range(cnt):
        try:
            name = g.get_plan_name_at_index(i)
            wsz = g.get_workspace_size_plan_at_index(i)
            w = torch.empty(max(wsz, 1), device="cuda", dtype=torch.uint8)
            pack = {Q: q, K: k, V: v, O: o}
            t = timeit(lambda: g.execute_plan_at_index(pack, w, i, handle=handle))
            err = (o.float() - ref.float()).abs().max().item()
            print(f"   plan {i} {name}: {t:.1f} us, max|d| vs torch {err:.1e}", flush=True)
        except Exception as e:   # noqa: BLE001
            print(f"   plan {i}: {type(e).__name__} {str(e)[:100]}", flush=True)
