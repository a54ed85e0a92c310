"""Summarise scripts/capture_tc_profiles.sh captures (gpurun_out/tc/*.raw.csv)
into the table of profiles/r2_tc_pipe.txt.

    python scripts/tc_pipe_summary.py gpurun_out/tc
"""
import csv
import glob
import os
import sys

M = {
    "us": "gpu__time_duration.sum",
    "tensor%": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "tmem%": "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "issue%": "sm__inst_issued.avg.pct_of_peak_sustained_active",
    "elig": "smsp__warps_eligible.avg.per_cycle_active",
    "dram_rd": "dram__bytes_read.sum",
    "dram_wr": "dram__bytes_write.sum",
    "conf": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "wav": "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
}


def num(v):
    try:
        return float(v.replace(",", ""))
    except ValueError:
        return float("nan")


def main(d):
    print(f"{'capture':16s} {'kernel':40s} {'us':>7s} {'tensor%':>8s} {'tmem%':>7s} {'issue%':>7s} "
          f"{'elig/cyc':>8s} {'DRAM MB':>8s} {'smem ld confl':>14s}")
    for f in sorted(glob.glob(os.path.join(d, "*.raw.csv"))):
        rows = list(csv.reader(open(f)))
        hdr, units, vals = rows[0], rows[1], rows[2]
        col = {h: i for i, h in enumerate(hdr)}
        scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        g = {k: num(vals[col[v]]) * (scale.get(units[col[v]], 1.0) if k.startswith("dram") else 1.0)
             if v in col else float("nan") for k, v in M.items()}
        us = g["us"] / 1e3 if units[col[M["us"]]] == "ns" else g["us"]
        name = vals[col["Kernel Name"]] if "Kernel Name" in col else "?"
        conf = 100.0 * g["conf"] / g["wav"] if g["wav"] else float("nan")
        print(f"{os.path.basename(f)[:-8]:16s} {name[:40]:40s} {us:7.1f} {g['tensor%']:8.1f} "
              f"{g['tmem%']:7.1f} {g['issue%']:7.1f} {g['elig']:8.2f} "
              f"{(g['dram_rd'] + g['dram_wr']) / 1e6:8.2f} {conf:13.0f} %")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/tc")
