"""DRAM traffic per entry point of one training step (bench.py roofline.traffic).

    # on the GPU box (one GPU), per entry point F:
    ncu --profile-from-start off --nvtx --nvtx-include "F/" \
        --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
        --cache-control none --clock-control none --csv --log-file gpurun_out/traffic_F.csv \
        python scripts/capture_traffic.py run --config C2
    python scripts/capture_traffic.py collect --config C2 gpurun_out/traffic_*.csv \
        > profiles/r2_traffic_C2.json

``run`` builds the bench Trainer, warms the captured step up, then runs ONE
eager step inside cudaProfilerStart/Stop with every qt_* ABI call wrapped in
an NVTX range of its name, so ncu's --nvtx-include selects exactly the
kernels one entry point launches.  ``collect`` sums dram__bytes_read.sum +
dram__bytes_write.sum per entry point and divides by its call count; the
JSON is stamped with the build digest of the sources it measured (bench.py
reports the number only while the digest matches).  --cache-control none:
the L2 state each kernel sees is the one the step leaves it.
"""

import argparse
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


class _Nvtx:
    def __init__(self, torch):
        self.torch = torch
        self.calls = {}

    def before(self, name, args):
        self.torch.cuda.nvtx.range_push(name)

    def after(self, name, args):
        self.torch.cuda.nvtx.range_pop()
        self.calls[name] = self.calls.get(name, 0) + 1


def run(cfg_name):
    import numpy as np
    import torch
    import bench
    import paper_1901_07988_b200 as P
    from paper_1901_07988_b200 import _native as N
    from paper_1901_07988_b200 import engine as E
    cfg = bench.CONFIGS[cfg_name]
    spec = getattr(E, cfg["builder"])()
    n = cfg["batch"]
    tr = P.Trainer(spec, n, mode="approx", bits=cfg["bits"], lr=0.1)
    rng = np.random.default_rng(0)
    tr.load_batch(rng.standard_normal((n,) + tuple(spec.input_shape)).astype(np.float32),
                  rng.integers(0, spec.num_classes, n))
    tr.capture()
    for _ in range(3):
        tr.step_device()
    torch.cuda.synchronize()
    hook = _Nvtx(torch)
    N.hook = hook
    torch.cuda.profiler.start()
    tr._body()
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    N.hook = None
    with open(os.path.join(ROOT, "gpurun_out", f"traffic_calls_{cfg_name}.json"), "w") as f:
        json.dump(hook.calls, f)


def collect(cfg_name, files):
    from paper_1901_07988_b200 import build as B
    with open(os.path.join(ROOT, "gpurun_out", f"traffic_calls_{cfg_name}.json")) as f:
        calls = json.load(f)
    fams = {}
    for path in files:
        fam = os.path.basename(path)[len("traffic_"):-len(".csv")]
        rows = []
        with open(path) as f:
            lines = [ln for ln in f if ln.startswith('"')]
        for r in csv.DictReader(lines):
            rows.append(r)
        by_id = {}
        for r in rows:
            k = r["ID"]
            d = by_id.setdefault(k, {"kernel": r["Kernel Name"], "read": 0.0, "write": 0.0,
                                     "ns": 0.0})
            v = float(r["Metric Value"].replace(",", ""))
            unit = r.get("Metric Unit", "")
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9,
                     "nsecond": 1, "usecond": 1e3, "msecond": 1e6}.get(unit, 1)
            if r["Metric Name"] == "dram__bytes_read.sum":
                d["read"] += v * scale
            elif r["Metric Name"] == "dram__bytes_write.sum":
                d["write"] += v * scale
            elif r["Metric Name"] == "gpu__time_duration.sum":
                d["ns"] += v * scale
        tot = sum(d["read"] + d["write"] for d in by_id.values())
        ncall = calls.get(fam, 0)
        fams[fam] = {"kernels": len(by_id), "calls": ncall, "dram_bytes": tot,
                     "dram_bytes_per_call": tot / ncall if ncall else None,
                     "serialized_ms": sum(d["ns"] for d in by_id.values()) * 1e-6}
    try:
        commit = subprocess.run(["git", "-C", ROOT, "rev-parse", "--short", "HEAD"],
                                capture_output=True, text=True).stdout.strip()
    except Exception:
        commit = None
    print(json.dumps({"config": cfg_name, "build_digest": B._digest(), "commit": commit,
                      "how": "ncu --nvtx-include <entry point>/ --metrics dram__bytes_read.sum,"
                             "dram__bytes_write.sum,gpu__time_duration.sum --cache-control none "
                             "--clock-control none over one eager step (scripts/capture_traffic.py)",
                      "families": fams}, indent=1))


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("mode", choices=["run", "collect"])
    ap.add_argument("--config", default="C2")
    ap.add_argument("files", nargs="*")
    a = ap.parse_intermixed_args()
    if a.mode == "run":
        run(a.config)
    else:
        collect(a.config, a.files)
