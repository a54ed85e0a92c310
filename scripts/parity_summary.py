"""Summarise gpurun_out/parity_<case>.json (tests/test_parity_gpu.py) into
the table committed as profiles/r2_parity_summary.txt."""
import glob
import json
import sys

files = sorted(glob.glob(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/parity_*.json"))
print(f"{'case':32s} {'L':>5s} {'fwd local max':>13s} {'bwd local max':>13s} {'logits err':>10s} "
      f"{'grad err (same tapes)':>21s} {'tol':>8s} {'flips own':>9s} {'flips vs oracle':>15s} "
      f"{'free-run grad err':>17s}")
for f in files:
    d = json.load(open(f))
    pl = d["per_layer"]
    own = sum(r.get("flips_vs_own_input", 0) for r in pl)
    el = sum(r.get("elements", 0) for r in pl)
    print(f"{d['case']:32s} {d['layers']:5d} {d['max_local_err']:13.2e} "
          f"{d.get('max_bwd_local_err', float('nan')):13.2e} {d['logits_err']:10.2e} "
          f"{d['worst_grad_err_identical_tapes']:21.2e} {d['grad_tol']:8.1e} {own:9d} "
          f"{d['total_flips_vs_oracle']:8d}/{el:<9d} {d['worst_grad_err_free_running']:14.2e}")
