"""Measure the dense i8 tensor-core peak of this B200 (the K3 roofline denominator).

cuBLASLt int8 x int8 -> int32 GEMM through torch._int_mm, M = N = K = 8192 (2*N^3 ops), best of 10
(burst) and back to back for 4 s (sustained), timed with CUDA events.  Writes profiles/i8_peak.json.
Run on the GPU box:  python tools/probes/i8_peak.py
"""
import json
import os
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    n = 8192
    a = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda")
    b = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda").t().contiguous().t()
    for _ in range(3):
        torch._int_mm(a, b)
    torch.cuda.synchronize()
    ops = 2.0 * n ** 3
    best = float("inf")
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch._int_mm(a, b)
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_end = time.time() + 4.0
    reps = 0
    e0.record()
    while time.time() < t_end:
        for _ in range(20):
            torch._int_mm(a, b)
        reps += 20
        torch.cuda.synchronize()
    e1.record()
    e1.synchronize()
    sus = ops * reps / (e0.elapsed_time(e1) / 1e3) / 1e12
    out = {"i8_tops_burst": ops / (best / 1e3) / 1e12, "i8_tops_sustained": sus,
           "how": "torch._int_mm (cuBLASLt int8 -> int32) 8192^3, 2*N^3 ops: best of 10 (burst), back to back "
                  "for 4 s (sustained), CUDA events",
           "gpu": torch.cuda.get_device_name(0), "torch": torch.__version__}
    print(json.dumps(out))
    with open(os.path.join(ROOT, "profiles", "i8_peak.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
