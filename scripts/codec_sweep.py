"""C5: codec kernel sweep.

    python scripts/codec_sweep.py [--out profiles/r1_codec_sweep_c5.txt] [--quick]

Times qt_quantize_pack (A2 -> packed K-bit codes + frozen constants,
codec.py:123-143) and qt_unpack_dequant (codes -> fp32 interval medians,
codec.py:146-156) over N in {32,128,256} x C in {16,64,256,1024} x
HW in {7^2,8^2,14^2,16^2,28^2,32^2,56^2} x K in {8,4,2}, with
x ~ 3 N(0,1) + 1, gamma ~ U(0.5, 2), beta ~ U(-1, 1).  Each rep is timed alone
with CUDA events on the launching stream after a 256 MiB L2 flush; the
algorithmic bytes are 4 + K/8 (quantize) and K/8 + 4 (dequantize) per element,
against the measured HBM peak.  Points whose working set is below 4x L2 are
marked (launch- and L2-bound, not roofline evidence)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1901_07988_b200 import codec

ap = argparse.ArgumentParser()
ap.add_argument("--out", default=None)
ap.add_argument("--quick", action="store_true", help="a 3x3x3x3 subset")
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()

dev = torch.device("cuda:0")
peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                    "MEASURED_PEAKS.json")))
hbm = float(peaks["hbm_gbs"])
l2 = torch.cuda.get_device_properties(dev).L2_cache_size
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
Ns, Cs, HWs, Ks = [32, 128, 256], [16, 64, 256, 1024], [7, 8, 14, 16, 28, 32, 56], [8, 4, 2]
if a.quick:
    Ns, Cs, HWs = [32, 256], [16, 256], [8, 32, 56]
gen = torch.Generator(device=dev).manual_seed(0)


def timed(fn):
    ts = []
    st = torch.cuda.current_stream()
    for _ in range(a.reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        fn()
        e1.record(st)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e-3)
    ts.sort()
    return ts[len(ts) // 2]


lines, rows = [], []
hdr = f"{'N':>4} {'C':>5} {'HW':>5} {'K':>2} {'MiB':>8} | {'quant GB/s':>10} {'frac':>5} | {'deq GB/s':>9} {'frac':>5} | note"
lines.append(hdr)
for K in Ks:
    for N in Ns:
        for C in Cs:
            for hw in HWs:
                numel = N * C * hw * hw
                if numel * 4 > 8 << 30:
                    continue
                x = torch.randn(N, C, hw, hw, device=dev, generator=gen).mul_(3).add_(1)
                gamma = torch.rand(C, device=dev, generator=gen) * 1.5 + 0.5
                beta = torch.rand(C, device=dev, generator=gen) * 2 - 1
                codes = torch.empty(codec.packed_nbytes(numel, K), dtype=torch.uint8, device=dev)
                t = codec.quantize(x, gamma, beta, K, codes_out=codes)
                out = torch.empty_like(x)
                tq = timed(lambda: codec.quantize(x, gamma, beta, K, codes_out=codes))
                td = timed(lambda: codec.dequantize(t, out=out))
                bq = numel * (4 + K / 8)
                bd = numel * (K / 8 + 4)
                gq, gd = bq / tq / 1e9, bd / td / 1e9
                big = numel * 4 >= 4 * l2
                rows.append(dict(N=N, C=C, HW=hw * hw, K=K, numel=numel, quant_gbs=gq,
                                 quant_frac=gq / hbm, dequant_gbs=gd, dequant_frac=gd / hbm,
                                 working_set_ge_4xL2=big))
                lines.append(f"{N:>4} {C:>5} {hw * hw:>5} {K:>2} {numel * 4 / 2**20:>8.1f} | "
                             f"{gq:>10.0f} {gq / hbm:>5.2f} | {gd:>9.0f} {gd / hbm:>5.2f} | "
                             f"{'' if big else '< 4xL2'}")
                del x, codes, t, out
big = [r for r in rows if r["working_set_ge_4xL2"]]


def med(v):
    v = sorted(v)
    return v[len(v) // 2] if v else None


summary = {"metric": "codec GB/s (C5 sweep)", "hbm_peak_gbs": hbm, "points": len(rows),
           "points_ge_4xL2": len(big),
           "quant_frac_median_ge_4xL2": med([r["quant_frac"] for r in big]),
           "dequant_frac_median_ge_4xL2": med([r["dequant_frac"] for r in big]),
           "quant_gbs_max": max(r["quant_gbs"] for r in rows),
           "dequant_gbs_max": max(r["dequant_gbs"] for r in rows)}
lines.append(json.dumps(summary))
text = "\n".join(lines)
print(text)
if a.out:
    with open(a.out, "w") as f:
        f.write(text + "\n")
