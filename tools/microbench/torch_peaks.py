"""cuBLAS reference throughput on this build's MLP layer shapes (context for the
roofline of the hand-written tcgen05 GEMMs) plus dense TF32 peak."""
import json, torch
def bench(fn, it=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(it): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / it
out = {}
for dt, name in [(torch.bfloat16, "bf16"), (torch.float32, "tf32")]:
    torch.backends.cuda.matmul.allow_tf32 = True
    a = torch.randn(8192, 8192, device="cuda", dtype=dt); b = torch.randn(8192, 8192, device="cuda", dtype=dt)
    ms = bench(lambda: a @ b)
    out[f"{name}_8192_tflops"] = 2 * 8192**3 / ms / 1e9
    for M, K, N in [(16384, 1600, 800), (131072, 1600, 800), (131072, 800, 400), (131072, 16, 1600)]:
        x = torch.randn(M, K, device="cuda", dtype=dt); w = torch.randn(N, K, device="cuda", dtype=dt)
        ms = bench(lambda: x @ w.t())
        out[f"{name}_{M}x{K}x{N}_tflops"] = 2 * M * K * N / ms / 1e9
print(json.dumps(out))
