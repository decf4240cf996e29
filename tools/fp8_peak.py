"""Measured dense FP8 tensor peak on this B200 (roofline denominator for the attention kernel).

torch._scaled_mm (cuBLASLt) e4m3 x e4m3 -> bf16 at 8192^3, best of 10 (burst) and back to back
for ~3 s (sustained), CUDA events.  Also an int8 torch._int_mm for the INT8 QK^T rate.
"""
import json
import time

import torch


def bench(fn, flops, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    burst = flops / (best * 1e-3) / 1e12
    n = 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.time()
    e0.record()
    while time.time() - t0 < 3.0:
        for _ in range(20):
            fn()
        n += 20
        torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    sustained = flops * n / (e0.elapsed_time(e1) * 1e-3) / 1e12
    return burst, sustained


def main():
    n = 8192
    a = torch.randn(n, n, device="cuda").to(torch.float8_e4m3fn)
    b = torch.randn(n, n, device="cuda").to(torch.float8_e4m3fn).t()
    one = torch.ones((), device="cuda")
    fp8 = bench(lambda: torch._scaled_mm(a, b, scale_a=one, scale_b=one, out_dtype=torch.bfloat16), 2.0 * n ** 3)
    ai = torch.randint(-127, 127, (n, n), device="cuda", dtype=torch.int8)
    bi = torch.randint(-127, 127, (n, n), device="cuda", dtype=torch.int8).t()
    try:
        i8 = bench(lambda: torch._int_mm(ai, bi), 2.0 * n ** 3)
    except Exception as e:  # noqa: BLE001
        i8 = (None, str(e))
    out = {"fp8_e4m3_tflops_burst": fp8[0], "fp8_e4m3_tflops_sustained": fp8[1],
           "int8_tops_burst": i8[0], "int8_tops_sustained": i8[1],
           "how": "torch._scaled_mm e4m3 8192^3 -> bf16 / torch._int_mm int8 8192^3; best of 10 (burst), "
                  "back to back ~3 s (sustained), CUDA events"}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
