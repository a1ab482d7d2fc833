"""cuBLAS ZGEMM / DGEMM throughput via torch (library baseline for the FP64 roofline)."""
import json, torch
def bench(dtype, m, n, k, reps=10):
    a = torch.randn(m, k, dtype=dtype, device="cuda"); b = torch.randn(k, n, dtype=dtype, device="cuda")
    for _ in range(3): a @ b
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    best = 1e30
    for _ in range(reps):
        e0.record(); a @ b; e1.record(); torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1))
    mult = 8 if dtype.is_complex else 2
    return mult * m * n * k / best / 1e9
out = {"dgemm_8192_tflops": bench(torch.float64, 8192, 8192, 8192),
       "zgemm_4096_tflops": bench(torch.complex128, 4096, 4096, 4096),
       # tall-skinny Gram shape of LOBPCG at n=128: (45 x 6.29M) @ (6.29M x 90)
       "zgemm_gram_45x90xK6.3M_tflops": bench(torch.complex128, 45, 90, 6291456, reps=5)}
print(json.dumps(out))
