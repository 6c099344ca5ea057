"""Same-box yardsticks (context only): cuBLAS ZGEMM/DGEMM via torch, HBM copy."""
import json, torch, time
def bench(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    best = 1e30
    for _ in range(reps):
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best
for n in (4096, 8192):
    a = torch.randn(n, n, dtype=torch.complex128, device="cuda"); b = torch.randn(n, n, dtype=torch.complex128, device="cuda")
    ms = bench(lambda: a @ b)
    print(json.dumps({"probe": "cublas_zgemm", "n": n, "tflops": 8 * n**3 / ms / 1e9}))
    a = torch.randn(n, n, dtype=torch.float64, device="cuda"); b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    ms = bench(lambda: a @ b)
    print(json.dumps({"probe": "cublas_dgemm", "n": n, "tflops": 2 * n**3 / ms / 1e9}))
# ZGEMM at a filter-like shape: 13000 x 13000 times 13000 x 624
n, k = 13000, 624
a = torch.randn(n, n, dtype=torch.complex128, device="cuda"); b = torch.randn(n, k, dtype=torch.complex128, device="cuda")
ms = bench(lambda: a @ b)
print(json.dumps({"probe": "cublas_zgemm_filter_shape", "n": n, "k": k, "tflops": 8 * n * n * k / ms / 1e9, "ms": ms}))
del a, b
x = torch.empty(2 * 1024**3 // 8, dtype=torch.float64, device="cuda"); y = torch.empty_like(x)
ms = bench(lambda: y.copy_(x))
print(json.dumps({"probe": "hbm_copy", "gbs": 2 * x.numel() * 8 / ms / 1e6}))
