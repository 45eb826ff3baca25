"""cuBLAS FP64 reference points (torch.matmul / torch.bmm in float64) for the roofline denominator."""
import json, torch
def t(fn, reps=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best
out = {}
a = torch.randn(8192, 8192, dtype=torch.float64, device="cuda"); b = torch.randn_like(a)
ms = t(lambda: a @ b); out["dgemm_8192_tflops"] = 2 * 8192**3 / ms / 1e9
for n, bt in [(256, 256), (256, 4096), (512, 64), (128, 2048)]:
    x = torch.randn(bt, n, n, dtype=torch.float64, device="cuda"); y = torch.randn_like(x)
    ms = t(lambda: torch.bmm(x, y)); out[f"bmm_{bt}x{n}^3_tflops"] = 2 * bt * n**3 / ms / 1e9
print(json.dumps(out))
