"""cuBLAS DGEMM (torch float64 matmul) throughput on this B200: the FP64 roofline denominator."""
import json, sys, time, torch

def best(n, reps=5):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    torch.matmul(a, b); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); c = torch.matmul(a, b); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3)
    return 2.0 * n ** 3 / min(ts) / 1e12, 2.0 * n ** 3 / (sum(ts) / len(ts)) / 1e12

out = {}
for n in [int(x) for x in sys.argv[1:]] or [4096, 8192, 16384]:
    bt, avg = best(n)
    out[n] = {"best_tflops": bt, "avg_tflops": avg}
    print(f"dgemm N={n}: best {bt:.2f} TF/s avg {avg:.2f} TF/s", flush=True)
print(json.dumps(out))
