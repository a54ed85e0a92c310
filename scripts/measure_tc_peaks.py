"""Dense tensor-core peaks for the roofline denominators, measured with the
MEASURED_PEAKS.json method (torch.matmul 8192^3, 2*N^3 FLOP: best of 10
(burst) and back to back for 4 s (sustained)), for the MMA kinds the conv
kernels issue: kind::tf32 (fp32 operands with TF32 tensor cores) and, as a
cross-check of the driver's number, kind::f16 (bf16).

    python scripts/measure_tc_peaks.py > profiles/r2_tc_peaks.json
"""

import json
import time

import torch


def rate(dtype, tf32):
    torch.backends.cuda.matmul.allow_tf32 = tf32
    n = 8192
    a = torch.randn(n, n, device="cuda", dtype=dtype)
    b = torch.randn(n, n, device="cuda", dtype=dtype)
    flop = 2 * n ** 3
    for _ in range(3):
        a @ b
    torch.cuda.synchronize()
    best = 0.0
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        a @ b
        e1.record()
        torch.cuda.synchronize()
        best = max(best, flop / (e0.elapsed_time(e1) * 1e-3) / 1e12)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.time()
    reps = 0
    e0.record()
    while time.time() - t0 < 4.0:
        for _ in range(20):
            a @ b
        reps += 20
        torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    sus = flop * reps / (e0.elapsed_time(e1) * 1e-3) / 1e12
    return best, sus


def main():
    tb, ts = rate(torch.float32, True)
    bb, bs = rate(torch.bfloat16, False)
    fb, fs = rate(torch.float32, False)
    print(json.dumps({
        "gpu": torch.cuda.get_device_name(0),
        "tf32_tflops": tb, "tf32_tflops_sustained": ts,
        "bf16_tflops": bb, "bf16_tflops_sustained": bs,
        "fp32_simt_tflops": fb, "fp32_simt_tflops_sustained": fs,
        "how": "torch.matmul 8192^3 (2 N^3 FLOP), CUDA events; best of 10 (burst) and back "
               "to back for 4 s (sustained); tf32 = fp32 operands with "
               "torch.backends.cuda.matmul.allow_tf32 (cuBLAS kind::tf32 tensor cores)",
        "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()),
    }, indent=1))


if __name__ == "__main__":
    main()
