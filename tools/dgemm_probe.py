"""cuBLAS DGEMM (torch.matmul fp64) throughput on the box: the library FP64 reference point."""
import json
import torch

def main():
    for n in (4096, 8192):
        a = torch.randn(n, n, dtype=torch.float64, device="cuda")
        b = torch.randn(n, n, dtype=torch.float64, device="cuda")
        for _ in range(2):
            torch.matmul(a, b)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = 1e30
        for _ in range(5):
            e0.record(); torch.matmul(a, b); e1.record(); torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        print(json.dumps({"probe": "cublas_dgemm", "n": n, "ms": best, "tflops": 2 * n**3 / best / 1e9}))

if __name__ == "__main__":
    main()
