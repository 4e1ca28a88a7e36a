"""Measure the dense int8 tensor-core peak on this B200 the way MEASURED_PEAKS.json measures bf16
(torch matmul 8192^3, best of 10, CUDA events). MEASURED_PEAKS.json has no int8 entry; the leaf
distance kernel's u8 path is judged against this number. Writes profiles/int8_peak.json."""
import json, sys, time
import torch

def bench(fn, iters=10):
    best = 1e30
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    for _ in range(iters):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best

N = 8192
a8 = torch.randint(-128, 127, (N, N), dtype=torch.int8, device="cuda")
b8 = torch.randint(-128, 127, (N, N), dtype=torch.int8, device="cuda").t().contiguous().t()
ms8 = bench(lambda: torch._int_mm(a8, b8))
ab = torch.randn(N, N, dtype=torch.bfloat16, device="cuda"); bb = torch.randn(N, N, dtype=torch.bfloat16, device="cuda")
msb = bench(lambda: ab @ bb)
out = {"int8_tops_burst": 2 * N**3 / ms8 / 1e9, "bf16_tflops_burst_same_run": 2 * N**3 / msb / 1e9,
       "how": "torch._int_mm int8 8192^3 and torch.matmul bf16 8192^3, best of 10 after 3 warmups, CUDA events",
       "gpu": torch.cuda.get_device_name(0)}
print(json.dumps(out))
if len(sys.argv) > 1:
    with open(sys.argv[1], "w") as f:
        json.dump(out, f, indent=1)
