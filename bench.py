#!/usr/bin/env python3
"""Benchmark of the B200 primitive layer (driver contract: one JSON line).

Headline workload (BASELINE.json configs[1]): one step =
  mapreduce f32 sum-of-squares over n = 2^30 floats  +  mapreduce i32 max over
  n = 2^30 ints, per GPU (weak scaling; at N > 1 the per-rank partials are
  exchanged with an NCCL all-gather and folded in rank order on the device).
metric = algorithmic HBM bytes / time (GB/s): 8 GiB read per GPU per step.
Inputs are 4 GiB each (>> 126 MB L2), so no L2 flush is needed between steps.

Also in the same line:
  roofline     the mapreduce kernel's achieved GB/s (CUDA events on its stream)
               against MEASURED_PEAKS.json hbm_gbs;
  e2e          the same metric through the reference-facing C-ABI Machine path
               (forge_write_bytes from pinned host memory + forge_mapreduce, whose
               result is read back to the host), host<->device copies timed;
  cpu_baseline the reference's own CPU implementation (the reference VM compiled
               from /root/reference into oracle/_ref/, Threads backend) on a
               bounded sample of the same workload, rank 0 only;
  breakdown    the other BASELINE configs on this GPU (scan C1/C3/C5-shard,
               gemv / gevm / min-plus C4, vcopy calibration).
`--impl reference` runs only the reference CPU arm.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

GIB = 1 << 30
N_C2 = 1 << 30


def measured_peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            d = json.loads(p.read_text())
            return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured"}
        except Exception:
            pass
    return {"hbm_gbs": 6650.0, "source": "fallback"}


def traffic_for(kernel_key: str):
    p = ROOT / "profiles" / "traffic.json"
    if p.exists():
        try:
            return json.loads(p.read_text()).get(kernel_key)
        except Exception:
            return None
    return None


class ClockSampler:
    """SM clock and clock-event (throttle) reasons sampled every 2 ms through
    NVML (the library behind nvidia-smi) while the timed region runs."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, device: int):
        self.device = device
        self.samples: list[tuple[int, int]] = []
        self.max_mhz = None
        self._stop = threading.Event()
        self._nvml = None

    def __enter__(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.device)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            get_reasons = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                nv.nvmlDeviceGetCurrentClocksThrottleReasons
            self._nvml = nv

            self._h, self._get_reasons = h, get_reasons

            def loop():
                while not self._stop.is_set():
                    self.sample_now()
                    time.sleep(0.002)

            self._t = threading.Thread(target=loop, daemon=True)
            self._t.start()
        except Exception:
            self._nvml = None
        return self

    def sample_now(self):
        """One synchronous sample (also called from the timed loop while the GPU is busy)."""
        if self._nvml is None:
            return
        try:
            nv = self._nvml
            self.samples.append((nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM), int(self._get_reasons(self._h))))
        except Exception:
            pass

    def __exit__(self, *exc):
        self._stop.set()
        if self._nvml is not None:
            self._t.join(timeout=2)

    def summary(self):
        if not self.samples:
            return None
        sms = sorted(s for s, _ in self.samples)
        mask = 0
        for _, r in self.samples:
            mask |= r
        reasons = sorted(name for bit, name in self.REASONS.items() if mask & bit)
        return {"sm_mhz": sms[len(sms) // 2], "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(self.samples), "source": "nvml (nvidia-smi backend), 2 ms"}


# ---------------------------------------------------------------------------
# reference CPU arm


def reference_arm(args, rank: int, world: int) -> None:
    if rank != 0:
        return
    import numpy as np

    from oracle import oracle as orc
    from oracle.ref import build_ref  # noqa: F401 (documents where the .so comes from)

    kind = "reference" if orc.ref_available() else "port"
    n = 1 << 20
    xs = orc.fill(1, n, 0x5EED0001)
    xi = orc.fill(6, n, 0x5EED0002)
    cores = min(os.cpu_count() or 2, 16)

    def step():
        t0 = time.perf_counter()
        if kind == "reference":
            orc.ref_mapreduce(1, xs, backend=orc.THREADS)
            orc.ref_mapreduce(6, xi, backend=orc.THREADS)
        else:
            orc.mapreduce(1, xs)
            orc.mapreduce(6, xi)
        return time.perf_counter() - t0

    for _ in range(args.warmup):
        step()
    times = [step() for _ in range(args.steps)]
    total = sum(times)
    byts = 2 * n * 4 * args.steps
    gbs = byts / total / 1e9
    line = {
        "metric": "mapreduce achieved HBM GB/s (f32 sum-of-squares + i32 max)", "impl": "reference",
        "value": gbs, "unit": "GB/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32+i32", "data": "synthetic",
        "config": {"workload": "C2 mapreduce f32 sum-of-squares + i32 max (bounded CPU sample)",
                   "sample_n_per_op": n},
        "cpu_baseline": {"value": gbs, "unit": "GB/s", "cores": cores, "kind": kind,
                         "sample": f"2 x 2^20-element mapreduce per step on the reference VM "
                                   f"Threads backend (clamp(hardware_concurrency,2,16) workers)"},
        "e2e": {"value": gbs, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline(seconds_budget: float = 12.0) -> dict:
    import numpy as np  # noqa: F401

    from oracle import oracle as orc
    kind = "reference" if orc.ref_available() else "port"
    n = 1 << 21
    xs = orc.fill(1, n, 0x5EED0001)
    xi = orc.fill(6, n, 0x5EED0002)
    total, reps, t_start = 0.0, 0, time.perf_counter()
    while reps < 3 or (time.perf_counter() - t_start < seconds_budget and reps < 20):
        t0 = time.perf_counter()
        if kind == "reference":
            orc.ref_mapreduce(1, xs, backend=orc.THREADS)
            orc.ref_mapreduce(6, xi, backend=orc.THREADS)
        else:
            orc.mapreduce(1, xs)
            orc.mapreduce(6, xi)
        total += time.perf_counter() - t0
        reps += 1
    gbs = 2 * n * 4 * reps / total / 1e9
    return {"value": gbs, "unit": "GB/s", "cores": min(os.cpu_count() or 2, 16) if kind == "reference" else 1,
            "kind": kind,
            "sample": f"{reps} x (f32 sum-of-squares + i32 max mapreduce over 2^21 elements each) on the "
                      f"reference VM Threads backend, {os.cpu_count()} host cores visible"}


# ---------------------------------------------------------------------------
# B200 arm


def forge_arm(args, rank: int, world: int, local_rank: int) -> None:
    import numpy as np  # noqa: F401
    import torch

    from paper_2603_18695_b200 import capi, dev
    from paper_2603_18695_b200 import forge as F

    # one process per GPU; FORGE_DIST_BACKEND=gloo lets a 1-GPU box run the
    # N>1 code path with every rank on cuda:0 (test only — NCCL is the product)
    local_rank = local_rank % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        backend = os.environ.get("FORGE_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group(backend)
    from paper_2603_18695_b200.sharded import _all_gather_bytes
    stream = torch.cuda.current_stream()
    n = args.elems
    ops = (capi.F32_SUMSQ, capi.I32_MAX)
    bufs = {}
    for i, op in enumerate(ops):
        bufs[op] = dev.empty(op, n)
        dev.fill_synthetic(op, bufs[op], n, seed=0x5EED0010 + i, index_base=rank * n)
    outs = {op: torch.zeros(16, dtype=torch.uint8, device="cuda") for op in ops}
    ssz = {op: F.op_info(op)["s_size"] for op in ops}
    final = {op: torch.zeros(16, dtype=torch.uint8, device="cuda") for op in ops}
    wss = {op: dev.Workspace() for op in ops}
    kern_ev = []  # (start, end) events around each mapreduce launch (roofline)

    def step(record=False):
        for op in ops:
            if record:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
            dev.mapreduce(op, bufs[op], n, outs[op], wss[op], stream=stream)
            if record:
                e1.record(stream)
                kern_ev.append((e0, e1))
            if world > 1:
                # partials exchange: sizeof(S) bytes per rank, folded in rank order on the device
                gath = _all_gather_bytes(outs[op][: ssz[op]], world)
                dev.fold(op, gath, world, final[op], stream=stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    sampler = ClockSampler(local_rank)
    with sampler:
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for _ in range(args.steps):
            step()
        t1.record(stream)
        # every step is queued: sample while the GPU works through them (an NVML
        # query takes milliseconds — never between enqueues, it would starve the GPU)
        sampler.sample_now()
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
    ms = t0.elapsed_time(t1)
    if dist:
        tt = torch.tensor([ms], device="cuda" if dist.get_backend() == "nccl" else "cpu")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    bytes_step = sum(n * F.op_info(op)["t_size"] for op in ops)
    value = world * bytes_step * args.steps / (ms * 1e-3) / 1e9

    elems_per_s = world * n * len(ops) * args.steps / (ms * 1e-3)

    # C5-style sharded exclusive scan on the same ranks (reduce-then-scan: ordered
    # shard reduce, all-gather of shard totals, rank-order fold, carry-seeded
    # local scan), 2^28 f32 per GPU, device-timed, max over ranks
    sharded_scan = None
    if not args.no_sharded_scan:
        from paper_2603_18695_b200 import sharded
        ns = 1 << 28
        xs = dev.empty(capi.F32_SUM, ns)
        dev.fill_synthetic(capi.F32_SUM, xs, ns, 0x5EED0C05, index_base=rank * ns)
        ys = dev.empty(capi.F32_SUM, ns, "S")
        be = sharded.DeviceBackend()
        for _ in range(3):
            sharded.sharded_scan(capi.F32_SUM, False, xs, ys, ns, backend=be)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 5
        e0.record(stream)
        for _ in range(reps):
            sharded.sharded_scan(capi.F32_SUM, False, xs, ys, ns, backend=be)
        e1.record(stream)
        torch.cuda.synchronize()
        sms = e0.elapsed_time(e1) / reps
        if dist:
            tt = torch.tensor([sms], device="cuda" if dist.get_backend() == "nccl" else "cpu")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            sms = float(tt.item())
        sharded_scan = {"workload": "exclusive scan f32 sum, 2^28 per GPU (C5 shape, weak scaling)",
                        "gbs": world * ns * 8 / (sms * 1e-3) / 1e9, "elems_per_s": world * ns / (sms * 1e-3),
                        "ms": sms, "hbm_bytes_per_gpu": 3 * ns * 4,
                        "note": "GB/s counts the algorithmic 8 B per element; the reduce-then-scan reads the input twice"}
        del xs, ys

    # roofline: the mapreduce kernel alone, events on its stream
    kern_ev.clear()
    for _ in range(3):
        step(record=True)
    torch.cuda.synchronize()
    kms = [a.elapsed_time(b) for a, b in kern_ev]
    kavg = sum(kms) / len(kms)
    peaks = measured_peaks()
    achieved = (n * 4) / (kavg * 1e-3) / 1e9
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / peaks["hbm_gbs"], "peak_source": peaks["source"],
                "frac_of_nominal_8tbs": achieved / 8000.0,
                "peak_note": "MEASURED_PEAKS hbm_gbs is a read+write copy (torch copy_); a read-only stream "
                             "exceeds it (frac > 1): the read roof measured by this kernel family is ~7.3 TB/s",
                "kernel": "mapreduce_kernel (f32 sumsq / i32 max, n=2^30)",
                "traffic": traffic_for("mapreduce_f32_sumsq_2^30"),
                "algorithmic_bytes_per_launch": n * 4, "avg_launch_ms": kavg}

    line = {
        "metric": "mapreduce achieved HBM GB/s (f32 sum-of-squares + i32 max)", "value": value, "unit": "GB/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32+i32",
        "data": "synthetic",
        "config": {"workload": "C2: mapreduce f32 sum-of-squares + i32 max, n=2^30 per GPU "
                               "(sharded mapreduce + NCCL all-gather of partials when N>1)",
                   "n_per_gpu": n, "global_n": n * world, "bytes_per_gpu_per_step": bytes_step,
                   "l2": "inputs 4 GiB each >> 126 MB L2; no flush needed",
                   "parallelism": f"shard{world}"},
        "elems_per_s": elems_per_s,
        "roofline": roofline,
        "gpu_launches": args.steps * len(ops) * (2 if world > 1 else 1),
        "clocks": sampler.summary(),
    }

    if sharded_scan is not None:
        line["sharded_scan"] = sharded_scan
    if not args.no_e2e:
        e2e = e2e_machine_path(args, n, ops, bufs, dist, world)
        if rank == 0:
            line["e2e"] = e2e
    if rank == 0 and world == 1 and not args.no_breakdown:
        line["breakdown"] = breakdown(args, peaks)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline()
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def e2e_machine_path(args, n, ops, dev_bufs, dist=None, world=1) -> dict:
    """The reference-facing call with HOST buffers on every rank: Machine.write_bytes
    from pinned memory (H2D) + forge_mapreduce (kernel + D2H of the S result); at
    N > 1 each rank's host result goes back to its GPU, the partials are
    all-gathered and folded in rank order, and the final value is read back.
    Whole-job bytes / the slowest rank's wall time (barriers on both sides)."""
    import numpy as np
    import torch

    from paper_2603_18695_b200 import dev
    from paper_2603_18695_b200 import forge as F
    from paper_2603_18695_b200.sharded import _all_gather_bytes

    m = F.Machine(torch.cuda.current_device())
    host = {}
    for op in ops:
        h = torch.empty(dev_bufs[op].numel(), dtype=torch.uint8, pin_memory=True)
        h.copy_(dev_bufs[op])
        host[op] = h
    bufs = {op: F.create_buffer(m, op, n) for op in ops}
    wss = {op: F.make_mapreduce_workspace(m, op) for op in ops}
    views = {op: F.View(bufs[op], 0, n, 1) for op in ops}
    final = torch.zeros(16, dtype=torch.uint8, device="cuda")

    def step():
        for op in ops:
            m.write_ptr(bufs[op], host[op].data_ptr(), host[op].numel())
            val, _ = F.mapreduce(m, F.make_semiring(op), views[op], wss[op])
            if world > 1:
                part = torch.from_numpy(np.array([val]).view(np.uint8).copy()).cuda()
                gath = _all_gather_bytes(part, world)
                dev.fold(op, gath, world, final)
                final.cpu()  # the job's result on the host

    for _ in range(max(1, min(args.warmup, 2))):
        step()
    k = max(2, min(args.steps, 5))
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(k):
        step()
    dt = time.perf_counter() - t0
    if dist:
        dist.barrier()
        tt = torch.tensor([dt], device="cuda" if dist.get_backend() == "nccl" else "cpu")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        dt = float(tt.item())
    byts = sum(host[op].numel() for op in ops)
    res = {"value": world * byts * k / dt / 1e9, "unit": "GB/s", "h2d_bytes_per_step": world * byts,
           "d2h_bytes_per_step": world * sum(F.op_info(op)["s_size"] for op in ops),
           "path": "forge_write_bytes(pinned host) + forge_mapreduce (host result)"
                   + (" + all-gather of partials, rank-order fold, D2H of the result" if world > 1 else ""),
           "steps": k}
    for op in ops:
        F.release(m, wss[op])
        m.destroy_buffer(bufs[op])
    m.close()
    return res


def _time_dev(fn, reps=5):
    import torch
    s = torch.cuda.current_stream()
    fn()
    torch.cuda.synchronize()
    evs = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        fn()
        b.record(s)
        evs.append((a, b))
    torch.cuda.synchronize()
    ts = sorted(x.elapsed_time(y) for x, y in evs)
    return ts[len(ts) // 2]


def breakdown(args, peaks) -> dict:
    import torch

    from paper_2603_18695_b200 import capi, dev

    out = {}
    peak = peaks["hbm_gbs"]

    def rec(name, byts, ms, elems=None, **kw):
        gbs = byts / (ms * 1e-3) / 1e9
        out[name] = {"gbs": round(gbs, 1), "ms": round(ms, 4), "frac": round(gbs / peak, 4), **kw}
        if elems:
            out[name]["elems_per_s"] = float(f"{elems / (ms * 1e-3):.4g}")

    ws = dev.Workspace()
    # vcopy calibration: 2 GiB copy
    nb = 2 * GIB
    a = torch.empty(nb, dtype=torch.uint8, device="cuda")
    b = torch.empty(nb, dtype=torch.uint8, device="cuda")
    rec("vcopy_2GiB", 2 * nb, _time_dev(lambda: dev.copy(a, b, nb)))
    rec("torch_copy_2GiB", 2 * nb, _time_dev(lambda: b.copy_(a)))
    del a, b
    # scans at n = 2^28
    n = 1 << 28
    for name, op, incl in (("scan_f32_sum_incl_2^28", capi.F32_SUM, True),
                           ("scan_f32_sum_excl_2^28", capi.F32_SUM, False),
                           ("scan_affine_f32_2^28", capi.AFFINE_F32, True),
                           ("scan_argmax_f32i32_2^28", capi.ARGMAX_F32I32, True),
                           ("scan_i32_sum_2^28", capi.I32_SUM, True)):
        src = dev.empty(op, n)
        dev.fill_synthetic(op, src, n, 0x5EED0003)
        dst = dev.empty(op, n, "S")
        sz = capi.load()  # noqa: F841
        ms = _time_dev(lambda: dev.scan(op, incl, src, dst, n, ws))
        from paper_2603_18695_b200.forge import op_info
        inf = op_info(op)
        rec(name, n * (inf["t_size"] + inf["s_size"]), ms, elems=n)
        del src, dst
    # C1: 2^20 scan (L2-resident, launch-bound)
    n1 = 1 << 20
    src = dev.empty(capi.F32_SUM, n1)
    dev.fill_synthetic(capi.F32_SUM, src, n1, 1)
    dst = dev.empty(capi.F32_SUM, n1, "S")
    rec("scan_f32_sum_2^20_C1", n1 * 8, _time_dev(lambda: dev.scan(capi.F32_SUM, True, src, dst, n1, ws), 20), elems=n1,
        note="8 MiB, L2-resident: one call per event pair, host launch latency included")
    # the same scan as a launch-bound loop captured in a CUDA graph (20 scans per replay)
    try:
        gstream = torch.cuda.Stream()
        gstream.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(gstream):
            for _ in range(3):
                dev.scan(capi.F32_SUM, True, src, dst, n1, ws)
        torch.cuda.current_stream().wait_stream(gstream)
        graph = torch.cuda.CUDAGraph()
        reps = 20
        with torch.cuda.graph(graph):
            for _ in range(reps):
                dev.scan(capi.F32_SUM, True, src, dst, n1, ws)
        ms = _time_dev(lambda: graph.replay(), 10) / reps
        rec("scan_f32_sum_2^20_C1_graph", n1 * 8, ms, elems=n1, note="20 scans per CUDA-graph replay; per-scan time")
    except Exception as e:  # noqa: BLE001 (report, do not fail the bench)
        out["scan_f32_sum_2^20_C1_graph"] = {"error": str(e)[:200]}
    # C4 matrices
    nn = 16384
    for name, op, fn in (("gevm_f32_16384^2 (ref matvec)", capi.MV_F32_PLUS_TIMES, dev.matvec),
                         ("gemv_f32_16384^2 (ref vecmat)", capi.MV_F32_PLUS_TIMES, dev.vecmat),
                         ("minplus_gevm_f32_16384^2", capi.MV_F32_MIN_PLUS, dev.matvec),
                         ("minplus_gemv_f32_16384^2", capi.MV_F32_MIN_PLUS, dev.vecmat)):
        A = dev.empty(op, nn * nn)
        dev.fill_synthetic(op, A, nn * nn, 5)
        x = dev.empty(op, nn)
        dev.fill_synthetic(op, x, nn, 6)
        y = dev.empty(op, nn, "S")
        ms = _time_dev(lambda: fn(op, A, nn, nn, x, y, ws))
        rec(name, nn * nn * 4 + 2 * nn * 4, ms, elems=nn * nn)
        del A, x, y
    # C2 extra: uf8 promotion
    src = dev.empty(capi.UF8_F32_SUM, N_C2)
    dev.fill_synthetic(capi.UF8_F32_SUM, src, N_C2, 7)
    outb = torch.zeros(16, dtype=torch.uint8, device="cuda")
    rec("mapreduce_uf8_f32_2^30", N_C2, _time_dev(lambda: dev.mapreduce(capi.UF8_F32_SUM, src, N_C2, outb, ws)),
        elems=N_C2)
    del src
    torch.cuda.empty_cache()
    # C5 at G = 1: n = 2^33 f32 (32 GiB in + 32 GiB out), exclusive scan and mapreduce;
    # the sharded path adds an order-preserving shard reduce (tests/test_gpu_fullsize.py)
    try:
        n5 = 1 << 33
        src = dev.empty(capi.F32_SUM, n5)
        dev.fill_synthetic(capi.F32_SUM, src, n5, 0x5EED0C05)
        dst = dev.empty(capi.F32_SUM, n5, "S")
        rec("scan_f32_sum_excl_2^33_C5_G1", n5 * 8, _time_dev(lambda: dev.scan(capi.F32_SUM, False, src, dst, n5, ws), 3),
            elems=n5)
        del dst
        o5 = torch.zeros(16, dtype=torch.uint8, device="cuda")
        rec("mapreduce_f32_sum_2^33_C5_G1", n5 * 4, _time_dev(lambda: dev.mapreduce(capi.F32_SUM, src, n5, o5, ws), 3),
            elems=n5)
        del src
    except Exception as e:  # noqa: BLE001 (e.g. a smaller GPU: report, do not fail the bench)
        out["C5_G1"] = {"error": str(e)[:200]}
    torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["forge", "reference"], default="forge")
    ap.add_argument("--elems", type=int, default=N_C2, help="elements per GPU per op")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-breakdown", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sharded-scan", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus if args.gpus == 1 else 1)))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        reference_arm(args, rank, world)
        return
    forge_arm(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
