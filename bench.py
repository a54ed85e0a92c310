"""Benchmark of the approximate-activation training step (BASELINE.json).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--config C2]

Default workload (BASELINE.json configs[1]): ResNet-164
CIFAR-10 shape, batch 128 per GPU (weak scaling), 4-bit approx tapes, one
full iteration per step = forward + softmax-xent + backward + (all-reduce)
+ momentum SGD, replayed from one CUDA graph.  Synthetic N(0,1) images, seed 0.

Prints ONE JSON line (rank 0).  ``value`` = whole-job images/s with inputs
resident in HBM; ``e2e`` = the same through the public Trainer.step() with
pinned-host H2D of every batch and a D2H of the loss inside the timed
region; ``roofline`` = the dominant kernel's algorithmic bytes / measured
time against MEASURED_PEAKS.json; ``cpu_baseline`` = the oracle port of the
reference (with the reference's own compiled C conv kernel from
oracle/_ref) timed on this host on a bounded sample.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "train images/sec + stored-activation bytes/sample at 4-bit, 1/2/4/8 B200"
CONFIGS = {
    "C1": dict(builder="make_residual_spec", batch=32, bits=4, classes=10,
               workload="C1 small CIFAR ResNet make_residual_spec(8,3,3), batch 32/GPU, 4-bit"),
    "C2": dict(builder="resnet164_spec", batch=128, bits=4, classes=10,
               workload="C2 ResNet-164 CIFAR-10 32x32, batch 128/GPU, 4-bit approx tapes"),
    "C3": dict(builder="resnet1001_spec", batch=128, bits=4, classes=100,
               workload="C3 ResNet-1001 CIFAR-100 32x32, batch 128/GPU, 4-bit approx tapes"),
    "C4": dict(builder="resnet152_spec", batch=64, bits=4, classes=1000,
               workload="C4 ResNet-152 224x224, batch 64/GPU, 4-bit approx tapes"),
}


def _peaks():
    """(HBM GB/s, bf16 dense TF/s sustained, tf32 dense TF/s sustained, kind).

    HBM and bf16 come from the driver-written MEASURED_PEAKS.json; the
    kind::tf32 rate from profiles/r2_tc_peaks.json, measured on this pool's
    B200s with the same method (torch.matmul 8192^3 back to back for 4 s,
    fp32 inputs with TF32 tensor cores: scripts/measure_tc_peaks.py)."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        hbm, bf16, kind = float(d["hbm_gbs"]), float(d["bf16_tflops_sustained"]), "measured"
    except Exception:
        hbm, bf16, kind = 6650.0, 1590.0, "fallback"
    try:
        with open(os.path.join(ROOT, "profiles", "r2_tc_peaks.json")) as f:
            tf32 = float(json.load(f)["tf32_tflops_sustained"])
    except Exception:
        tf32, kind = bf16 / 2, kind + " (tf32 = bf16/2 fallback)"
    return hbm, bf16, tf32, kind


# MMA issue model of each conv entry point: the
# forward and data-gradient GEMMs run 3xTF32 (three kind::tf32 passes per
# useful FLOP); the weight gradient from 4-bit codes runs kind::f16 with g
# split into three bf16 pieces (three passes), GENERIC tapes 3xTF32.
TC_PASSES = {"qt_conv_forward": ("tf32", 3), "qt_conv_dgrad": ("tf32", 3),
             "qt_conv_wgrad": ("bf16", 3)}


def _traffic(entry, cfg_name):
    """DRAM bytes per call of ``entry`` (dram__bytes_read.sum +
    dram__bytes_write.sum over every kernel launched inside the entry
    point's NVTX range in one step, scripts/capture_traffic.py under ncu),
    if the committed capture was taken from the current sources (build
    digest match); else None."""
    try:
        from paper_1901_07988_b200 import build as B
        with open(os.path.join(ROOT, "profiles", f"r2_traffic_{cfg_name}.json")) as f:
            t = json.load(f)
    except Exception:
        return None, "no capture"
    fam = t.get("families", {}).get(entry)
    if fam is None:
        return None, "entry point not in capture"
    if t.get("build_digest") != B._digest():
        return None, f"stale capture (digest {t.get('build_digest')})"
    return fam["dram_bytes_per_call"], "ncu capture of the current build"


# ------------------------------------------------------------ cost model

def _geo(args, off):
    n, ci, h, w, co, kh, kw, s, p = (int(args[off + i]) for i in range(9))
    oh = (h + 2 * p - kh) // s + 1
    ow = (w + 2 * p - kw) // s + 1
    return n, ci, h, w, co, kh, kw, oh, ow


def algo_cost(name, a):
    """(algorithmic HBM bytes, useful FLOPs) of one qt_* call."""
    if name in ("qt_bn_stats", "qt_bn_stats_prep"):
        return 4 * a[1] * a[2] * a[3], 0
    if name == "qt_bn_forward_fused":
        numel = a[1] * a[2] * a[3]
        b = 8 * numel + ((a[8] * numel + 7) // 8 if a[8] else 0) + (4 * numel if a[20] else 0)
        return b, 0
    if name == "qt_bn_relu_forward":
        numel = a[1] * a[2] * a[3]
        b = 4 * numel + (4 * numel if a[11] else 0) + (4 * numel if a[12] else 0)
        b += (a[10] * numel + 7) // 8 if a[10] else 0
        return b, 0
    if name == "qt_conv_forward":
        n, ci, h, w, co, kh, kw, oh, ow = _geo(a, 3)
        b = 4 * (n * ci * h * w + n * co * oh * ow + co * ci * kh * kw)
        if a[12]:
            b += 4 * n * int(a[13]) * oh * ow
        return b, 2 * n * oh * ow * co * ci * kh * kw
    if name == "qt_conv_dgrad":
        n, ci, h, w, co, kh, kw, oh, ow = _geo(a, 3)
        return (4 * (n * co * oh * ow + n * ci * h * w + co * ci * kh * kw),
                2 * n * oh * ow * co * ci * kh * kw)
    if name == "qt_conv_wgrad":
        n, ci, h, w, co, kh, kw, oh, ow = _geo(a, 4)
        tape = a[1]
        act = n * ci * h * w
        ab = (tape.bits * act + 7) // 8 if (tape.codes and not a[2]) else 4 * act
        return (4 * n * co * oh * ow + ab + 8 * co * ci * kh * kw,
                2 * n * oh * ow * co * ci * kh * kw)
    if name in ("qt_bn_backward_reduce", "qt_bn_backward_apply"):
        tape = a[1]
        numel = a[2] * a[3] * a[4] * (a[5] if name == "qt_bn_backward_apply" else 1)
        tb = (tape.bits * numel + 7) // 8 if tape.codes else 4 * numel
        b = 4 * numel + tb + (4 * numel if name == "qt_bn_backward_apply" else 0)
        if name == "qt_bn_backward_apply" and a[10]:
            b += 4 * numel // (int(a[12]) ** 2)
        return b, 0
    if name == "qt_copy":
        return 8 * a[2], 0
    if name == "qt_sgd":
        return 16 * a[3], 0
    return 0, 0


class CallRecorder:
    """_native hook: records every qt_* call (name, ctypes args) of one step."""

    def __init__(self):
        self.calls = []

    def before(self, name, args):
        pass

    def after(self, name, args):
        self.calls.append((name, args))


def family_times(torch, N, calls, reps=5):
    """Per-entry-point device time of one step, measured live: all of a
    step's calls of one qt_* entry point are captured (same arguments, same
    order) into a CUDA graph and replayed on the launching stream between
    CUDA events, so the time is kernel time, not host launch overhead."""
    agg = {}
    for name, args in calls:
        d = agg.setdefault(name, {"ms": 0.0, "launches": 0, "bytes": 0, "flops": 0, "calls": []})
        b, f = algo_cost(name, args)
        d["launches"] += 1
        d["bytes"] += b
        d["flops"] += f
        d["calls"].append(args)
    s = torch.cuda.Stream()
    for name, d in agg.items():
        fn = getattr(N.lib(), name)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                for args in d["calls"]:
                    fn(*args, N.stream())
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(s)
            for _ in range(reps):
                g.replay()
            e1.record(s)
        torch.cuda.synchronize()
        d["ms"] = e0.elapsed_time(e1) / reps
        del d["calls"]
    return agg


class _FamilyEvents:
    """_native hook: external timing events around every call of one entry
    point, recorded on the stream the call is launched on (inside a CUDA
    graph capture they become event-record nodes)."""

    def __init__(self, torch, family):
        self.torch, self.family, self.pairs = torch, family, []

    def before(self, name, args):
        if name == self.family:
            ev = self.torch.cuda.Event(enable_timing=True, external=True)
            ev.record()
            self.pairs.append([ev, None])

    def after(self, name, args):
        if name == self.family:
            ev = self.torch.cuda.Event(enable_timing=True, external=True)
            ev.record()
            self.pairs[-1][1] = ev


def concurrent_family_ms(torch, N, tr, family, reps=3):
    """Device time per step of ``family`` inside the real captured step
    (the weight gradients overlapping the data-gradient chain): one more
    capture of the step with external events around each of its calls,
    replayed; the per-launch durations are summed."""
    try:
        hook = _FamilyEvents(torch, family)
        g = torch.cuda.CUDAGraph()
        cs = torch.cuda.Stream()
        cs.wait_stream(torch.cuda.current_stream())
        N.hook = hook
        try:
            with torch.cuda.stream(cs):
                with torch.cuda.graph(g, stream=cs):
                    tr._body()
        finally:
            N.hook = None
        torch.cuda.synchronize()
        tot = 0.0
        for _ in range(reps):
            g.replay()
            torch.cuda.synchronize()
            tot += sum(a.elapsed_time(b) for a, b in hook.pairs)
        del g
        return tot / reps
    except Exception as e:          # measurement aid only; never fails the bench
        print(f"concurrent timing unavailable: {e}", file=sys.stderr)
        return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        sm.sort()
        med = sm[len(sm) // 2] if sm else None
        return {"sm_mhz": med, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------- CPU baseline

def _cpu_worker(cfg_name, batch, steps, warmup, q, budget_s=None, seed=0):
    os.environ["OMP_NUM_THREADS"] = "1"
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    import numpy as np
    import oracle as O
    from paper_1901_07988_b200 import engine as E
    c = CONFIGS[cfg_name]
    spec = getattr(E, c["builder"])().to_json()
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((batch,) + tuple(spec["input_shape"])).astype(np.float32)
    y = rng.integers(0, spec["num_classes"], batch)
    params = O.init_params(spec, 0)
    times = []
    t_start = time.perf_counter()
    for i in range(warmup + steps):
        t0 = time.perf_counter()
        O.train_step(spec, params, x, y, "approx", c["bits"])
        if i >= warmup:
            times.append(time.perf_counter() - t0)
            # time-bounded sample: at least one timed step, then stop once
            # the budget is spent
            if budget_s is not None and time.perf_counter() - t_start > budget_s:
                break
    q.put(times)


def cpu_reference(cfg_name, batch, steps, warmup, procs, budget_s=None):
    """Oracle port (+ reference C kernel) on `procs` single-thread processes,
    each a shard of `batch` images (distinct data per process); returns
    (aggregate images/s, median step seconds)."""
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_cpu_worker, args=(cfg_name, batch, steps, warmup, q, budget_s, r))
          for r in range(procs)]
    for p in ps:
        p.start()
    res = [q.get() for _ in ps]
    for p in ps:
        p.join()
    med = [sorted(t)[len(t) // 2] for t in res]
    return sum(batch / m for m in med), sorted(med)[len(med) // 2]


# ------------------------------------------------------------------ main

def _comm_info(torch, tr, group, world):
    """Data-parallel exchange of this run: backend, rank count (from the
    process group itself), NCCL version, gradient buckets."""
    if group is None:
        return {"backend": None, "nranks": 1, "allreduce": "none (single GPU)"}
    import torch.distributed as dist
    ver = torch.cuda.nccl.version()
    info = {"backend": dist.get_backend(group), "nranks": dist.get_world_size(group),
            "nranks_ok": dist.get_world_size(group) == world,
            "nccl_version": ".".join(map(str, ver)) if isinstance(ver, tuple) else str(ver),
            "grad_bytes": tr.params.grads.numel() * 4}
    if tr.buckets is not None:
        info.update(allreduce="bucketed AVG on a comm stream, overlapped with backward, in-graph",
                    buckets=len(tr.buckets.buckets) + 1,
                    bucket_bytes=[(b[2] - b[1]) * 4 for b in tr.buckets.buckets])
    else:
        info.update(allreduce="one AVG over the whole slab between two graph replays")
    return info


def _spawn_ranks(n):
    """``bench.py --gpus N`` without a launcher: re-run this command under
    torch.distributed.run with N ranks on this node (127.0.0.1 rendezvous);
    NCCL prints its communicator-init lines (NCCL_DEBUG=INFO, INIT subsystem)
    to stderr so the rank count can be checked.  Exits with the launcher's
    status."""
    import socket
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd, env=env))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C2", choices=sorted(CONFIGS))
    ap.add_argument("--bits", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-batch", type=int, default=0,
                    help="reference arm: images per process (0: the config batch / cores); "
                         "cpu_baseline leg: 4")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    bits = args.bits or cfg["bits"]
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        if args.impl != "reference":
            import torch
            if torch.cuda.device_count() < args.gpus:
                print(json.dumps({"error": f"--gpus {args.gpus} but {torch.cuda.device_count()} "
                                           f"GPU(s) visible"}), flush=True)
                sys.exit(2)
        _spawn_ranks(args.gpus)            # re-exec under torchrun: one rank per GPU
        return
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world != args.gpus:
        print(json.dumps({"error": f"--gpus {args.gpus} but WORLD_SIZE={world}: launch one "
                                   f"rank per GPU"}), flush=True)
        sys.exit(2)

    if args.impl == "reference":
        if rank != 0:
            return
        procs = max(1, len(os.sched_getaffinity(0)))
        steps = max(1, args.steps)
        # the config's per-GPU batch per step, sharded over the host's cores
        # (one single-thread process per core, local BN per shard as the
        # data-parallel GPU path); time-bounded so the run ends in minutes
        shard = max(1, -(-cfg["batch"] // procs)) if args.cpu_batch <= 0 else args.cpu_batch
        budget = 120.0
        ips, med = cpu_reference(args.config, shard, steps, max(0, min(args.warmup, 1)), procs,
                                 budget_s=budget)
        line = {
            "metric": METRIC, "value": ips, "unit": "images/s", "impl": "reference",
            "n_gpus": args.gpus, "steps": steps, "warmup": args.warmup,
            "ms_per_step": med * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32 (f64 accumulation)", "data": "synthetic",
            "config": {"workload": cfg["workload"], "images_per_step": shard * procs,
                       "batch_per_process": shard, "processes": procs},
            "cpu_baseline": {"value": ips, "unit": "images/s", "cores": procs, "kind": "port",
                             "sample": f"{procs} single-thread processes x batch {shard} = "
                                       f"{shard * procs} images per step ({args.config} spec, "
                                       f"the config's batch {cfg['batch']} sharded over the "
                                       f"cores), up to {steps} steps or {budget:.0f} s"},
            "e2e": {"value": ips, "unit": "images/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
        }
        print(json.dumps(line), flush=True)
        return

    import numpy as np
    import torch
    import paper_1901_07988_b200 as P
    from paper_1901_07988_b200 import _native as N
    from paper_1901_07988_b200 import dist as D
    from paper_1901_07988_b200 import engine as E

    group = None
    local = 0
    if world > 1:
        rank, world, local = D.init_from_env("nccl")
        group = torch.distributed.group.WORLD
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    spec = getattr(E, cfg["builder"])()
    n = cfg["batch"]
    tr = P.Trainer(spec, n, mode="approx", bits=bits, lr=0.1, momentum=0.9,
                   weight_decay=2e-4 if args.config != "C4" else 1e-4, seed=0, device=dev,
                   process_group=group)
    if group is not None:
        D.broadcast_(tr.params.values, 0)
    rng = np.random.default_rng(rank)
    # the host batch lives in pinned memory (the e2e contract's source); the
    # Trainer copies it to the device directly, no staging memcpy
    x_host = torch.from_numpy(rng.standard_normal((n,) + tuple(spec.input_shape)).astype(np.float32)).pin_memory()
    y_host = torch.from_numpy(rng.integers(0, spec.num_classes, n).astype(np.int64)).pin_memory()
    tr.load_batch(x_host, y_host)
    tr.capture()

    # launches per step: count one eager step
    c0 = N.launch_count[0]
    tr._body()
    launches_per_step = N.launch_count[0] - c0
    torch.cuda.synchronize()

    for _ in range(max(3, args.warmup)):
        tr.step_device()
    torch.cuda.synchronize()

    def barrier():
        if group is not None:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    clocks = ClockSampler(local)
    clocks.start()
    barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        tr.step_device()
    e1.record()
    barrier()
    ms = e0.elapsed_time(e1) / args.steps
    ms = D.max_over_ranks(ms, group, dev)

    # end to end through the public API: host batch -> H2D -> step -> D2H loss
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        tr.step(x_host, y_host)
    barrier()
    e2e_s = (time.perf_counter() - t0) / args.steps
    e2e_s = D.max_over_ranks(e2e_s, group, dev)
    clk = clocks.stop()

    # per-entry-point device time (graph replay of each entry point's calls
    # of one step, CUDA events on the launching stream) -> dominant kernel
    # and its roofline; done last because replaying one family alone
    # disturbs the model state
    # (the calls are recorded while capturing one more graph of the step, so
    # every temporary they point at lives in that graph's memory pool for
    # as long as `hold` exists)
    rec = CallRecorder()
    hold = torch.cuda.CUDAGraph()
    cs = torch.cuda.Stream()
    cs.wait_stream(torch.cuda.current_stream())
    N.hook = rec
    with torch.cuda.stream(cs):
        with torch.cuda.graph(hold, stream=cs):
            tr._body()
    N.hook = None
    torch.cuda.synchronize()
    # replay each family with the launch shapes of the step (the side-stream
    # SM partition is scoped to network_backward, so set it here as well)
    ws = tr.pool.cache[("ws", id(spec), n)]
    prev = N.query("qt_set_concurrent_backward", int(ws.side is not None))
    agg = family_times(torch, N, rec.calls)
    N.query("qt_set_concurrent_backward", prev)
    del hold
    hbm, bf16, tf32, peak_kind = _peaks()
    total_ms = sum(d["ms"] for d in agg.values())
    top = max(agg.items(), key=lambda kv: kv[1]["ms"])
    name, d = top
    conc_ms = concurrent_family_ms(torch, N, tr, name)

    def tc_time(nm, dd):
        kind, passes = TC_PASSES.get(nm, ("bf16", 1))
        return passes * dd["flops"] / ((tf32 if kind == "tf32" else bf16) * 1e12)

    if d["flops"] and tc_time(name, d) > d["bytes"] / (hbm * 1e9):
        kind, passes = TC_PASSES.get(name, ("bf16", 1))
        pk = (tf32 if kind == "tf32" else bf16) / passes
        achieved = d["flops"] / (d["ms"] * 1e-3) / 1e12
        roof = {"bound": "tensor", "achieved": achieved, "peak": pk, "unit": "TFLOP/s",
                "frac": achieved / pk,
                "peak_note": f"useful FLOP/s: {kind} dense sustained / {passes} split passes"}
    else:
        achieved = d["bytes"] / (d["ms"] * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                "frac": achieved / hbm}
    traffic, traffic_src = _traffic(name, args.config)
    per = d["bytes"] / d["launches"] if d["launches"] else None
    roof.update({"kernel": name, "launches_per_step": d["launches"],
                 "ms_per_step_isolated": d["ms"],
                 "ms_per_step_concurrent": conc_ms,
                 "timing": "isolated: the family's calls of one step replayed alone from a CUDA "
                           "graph (step launch shapes); concurrent: sum of per-launch durations "
                           "inside the captured step (external CUDA events on the launching "
                           "stream)",
                 "share_of_step": d["ms"] / total_ms if total_ms else None,
                 "traffic": traffic, "traffic_source": traffic_src,
                 "traffic_over_algorithmic": traffic / per if (traffic and per) else None,
                 "peak_kind": peak_kind, "algorithmic_bytes_per_launch": per})
    if conc_ms:
        a_c = (d["bytes"] / (conc_ms * 1e-3) / 1e9) if roof["bound"] == "hbm" else \
            d["flops"] / (conc_ms * 1e-3) / 1e12
        roof["frac_concurrent"] = a_c / roof["peak"]
    # step roofline: every launch at its own bound (HBM or tensor), summed
    step_roof_ms = 0.0
    for nm, dd in agg.items():
        step_roof_ms += max(dd["bytes"] / (hbm * 1e9), tc_time(nm, dd)) * 1e3
    kernels = sorted(({"kernel": k, "ms": v["ms"], "launches": v["launches"],
                       "GBps": v["bytes"] / (v["ms"] * 1e-3) / 1e9 if v["ms"] else None,
                       "TFps": v["flops"] / (v["ms"] * 1e-3) / 1e12 if v["ms"] and v["flops"] else None}
                      for k, v in agg.items()), key=lambda r: -r["ms"])[:8]

    rep = E.memory_report(spec, (n,) + tuple(spec.input_shape), mode="approx", bits=bits)
    rep_exact = E.memory_report(spec, (n,) + tuple(spec.input_shape), mode="exact", bits=None)
    images = n * world
    value = images / (ms * 1e-3)
    line = {
        "metric": METRIC, "value": value, "unit": "images/s", "n_gpus": world,
        "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic N(0,1) images, seed 0, random-init weights",
        "config": {"workload": cfg["workload"], "global_batch": images, "per_gpu_batch": n,
                   "bits": bits, "mode": "approx", "parallelism": f"dp{world}",
                   "l2": f"step working set > L2 (tape arena {tr.arena.code_arena_bytes >> 20} MiB, "
                         f"{len(spec.layers)} layers streamed per step)"},
        "stored_activation_bytes_per_sample": rep.persistent_tape_bytes // n,
        "exact_activation_bytes_per_sample": rep_exact.persistent_tape_bytes // n,
        "activation_reduction": rep_exact.persistent_tape_bytes / rep.persistent_tape_bytes,
        "e2e": {"value": images / e2e_s, "unit": "images/s",
                "h2d_bytes_per_step": tr.h2d_bytes, "d2h_bytes_per_step": tr.d2h_bytes},
        "gpu_launches": launches_per_step * args.steps,
        "comm": _comm_info(torch, tr, group, world),
        "roofline": roof,
        "step_roofline": {"ms": step_roof_ms, "frac": step_roof_ms / ms},
        "kernels": kernels,
        "clocks": clk,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        procs = 1
        cb = args.cpu_batch if args.cpu_batch > 0 else 4
        ips, med = cpu_reference(args.config, cb, 2, 1, procs)
        line["cpu_baseline"] = {"value": ips, "unit": "images/s", "cores": procs, "kind": "port",
                                "sample": f"1 warm-up + 2 steps at batch {cb} of the "
                                          f"{args.config} network, oracle port + reference C "
                                          f"conv kernel, 1 thread ({med:.1f} s/step)"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if group is not None:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
