"""Measure the TF32-dense and FP64 tensor peaks on the box.

Same method as the driver's MEASURED_PEAKS.json: torch.matmul on N^3 operands,
best of 10 timed with CUDA events (2 N^3 flops per product).  Writes one JSON
line; the committed copy lives in profiles/peaks_tf32_fp64.json."""
import json
import sys

import torch


def best(fn, n, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / 1e3)
    return 2 * n ** 3 / min(ts) / 1e12


def main():
    out = {"gpu": torch.cuda.get_device_name(0)}
    n = 8192
    a = torch.randn(n, n, device="cuda")
    b = torch.randn(n, n, device="cuda")
    torch.backends.cuda.matmul.allow_tf32 = True
    out["tf32_tflops"] = best(lambda: a @ b, n)
    torch.backends.cuda.matmul.allow_tf32 = False
    out["fp32_simt_tflops"] = best(lambda: a @ b, n)
    n2 = 8192
    ad = torch.randn(n2, n2, device="cuda", dtype=torch.float64)
    bd = torch.randn(n2, n2, device="cuda", dtype=torch.float64)
    out["fp64_tflops"] = best(lambda: ad @ bd, n2, reps=5)
    ac = torch.randn(4096, 4096, device="cuda", dtype=torch.complex128)
    bc = torch.randn(4096, 4096, device="cuda", dtype=torch.complex128)
    # ZGEMM: 8 real flops per complex MAC
    out["zgemm_tflops"] = best(lambda: ac @ bc, 4096, reps=5) * 4
    ah = torch.randn(n, n, device="cuda", dtype=torch.float16)
    bh = torch.randn(n, n, device="cuda", dtype=torch.float16)
    out["fp16_tflops"] = best(lambda: ah @ bh, n)
    out["how"] = "torch.matmul N=8192 (ZGEMM N=4096, x4 for complex), best of 10 (5 for fp64), CUDA events"
    print(json.dumps(out))


if __name__ == "__main__":
    sys.exit(main())
