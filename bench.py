#!/usr/bin/env python3
"""Benchmark of the B200 primitive layer (driver contract: one JSON line).

metric (BASELINE.json): scan/mapreduce/matvec achieved HBM GB/s.  One STEP is
the composite of BASELINE's single-GPU configs, per GPU (weak scaling: every
rank owns one shard of each global problem):

  C2  mapreduce f32 sum-of-squares, n = 2^30      (4 GiB read)
  C2  mapreduce i32 max,            n = 2^30      (4 GiB read)
  C5  exclusive scan f32 sum,       n = 2^28      (1 GiB read + 1 GiB written)
  C3  inclusive scan Affine{f32 a,b} 2x2 affine-map composition, n = 2^28 (2 + 2 GiB)
  C3  inclusive scan ArgMax{f32 v, i32 i},       n = 2^28 (2 + 2 GiB)
  C4  gevm f32 16384 x 16384 (reference matvec)  (1 GiB)
  C4  gemv f32 16384 x 16384 (reference vecmat)  (1 GiB)
  C4  min-plus gevm 16384 x 16384                (1 GiB)

At N > 1 the mapreduces all-gather the per-rank partials and fold them in rank
order, the scans are GLOBAL scans of the rank-ordered concatenation
(reduce-then-scan: ordered shard reduce, all-gather of shard totals, rank-order
fold, carry-seeded local scan), gevm owns a column block and gemv a row block of
the global matrix (no collective).  value = whole-job algorithmic bytes / the
slowest rank's device time (CUDA events, max over ranks).  Inputs are >> the
126 MB L2 (21 GiB touched per step per GPU), so no flush is needed.

Also in the line: per-component GB/s from the same timed region; `roofline`
of the dominant kernel (largest share of the step) and of every kernel;
`c5` = BASELINE C5 itself (n = 2^33 f32 GLOBAL, strong scaling: 2^33/N per
GPU, sharded exclusive scan + sharded mapreduce); `e2e` = the same composite
through the public API with host buffers (pinned H2D of every input, D2H of
every result); `cpu_baseline` = the reference's own CPU implementation (the
reference VM, Threads backend, compiled from /root/reference into
oracle/_ref/) on a bounded sample of the same composite, per primitive.
`--impl reference` runs only that CPU arm.
`--gpus N` without WORLD_SIZE re-launches itself under torch.distributed.run.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

GIB = 1 << 30
N_MR = 1 << 30
N_SCAN = 1 << 28
N_MAT = 16384
N_C5 = 1 << 33

METRIC = "scan/mapreduce/matvec achieved HBM GB/s"


def measured_peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            d = json.loads(p.read_text())
            return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured (MEASURED_PEAKS.json hbm_gbs)"}
        except Exception:
            pass
    return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


def traffic_table() -> dict:
    """ncu dram__bytes_read.sum + dram__bytes_write.sum per launch, from the
    committed full captures (profiles/r02/traffic.json)."""
    for p in (ROOT / "profiles" / "r02" / "traffic.json", ROOT / "profiles" / "traffic.json"):
        if p.exists():
            try:
                return json.loads(p.read_text())
            except Exception:
                pass
    return {}


class ClockSampler:
    """SM clock and clock-event (throttle) reasons sampled through NVML (the
    library behind nvidia-smi) while the timed region runs."""

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
            self._nvml, self._h, self._get_reasons = nv, h, get_reasons

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
        if self._nvml is None:
            return
        try:
            nv = self._nvml
            self.samples.append((nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM),
                                 int(self._get_reasons(self._h))))
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
# the composite workload


def component_specs():
    """(name, kind, op, inclusive, n or (rows, cols), algorithmic bytes per GPU)."""
    from paper_2603_18695_b200 import capi
    from paper_2603_18695_b200.forge import op_info

    def sz(op, which="T"):
        return op_info(op)["t_size" if which == "T" else "s_size"]

    mat_bytes = N_MAT * N_MAT * 4 + 2 * N_MAT * 4
    return [
        ("mapreduce_f32_sumsq", "mapreduce", capi.F32_SUMSQ, None, N_MR, N_MR * sz(capi.F32_SUMSQ)),
        ("mapreduce_i32_max", "mapreduce", capi.I32_MAX, None, N_MR, N_MR * sz(capi.I32_MAX)),
        ("scan_f32_sum_excl", "scan", capi.F32_SUM, False, N_SCAN, N_SCAN * (sz(capi.F32_SUM) + 4)),
        ("scan_affine_f32", "scan", capi.AFFINE_F32, True, N_SCAN, N_SCAN * 2 * sz(capi.AFFINE_F32)),
        ("scan_argmax_f32i32", "scan", capi.ARGMAX_F32I32, True, N_SCAN, N_SCAN * 2 * sz(capi.ARGMAX_F32I32)),
        ("gevm_f32", "matvec", capi.MV_F32_PLUS_TIMES, None, (N_MAT, N_MAT), mat_bytes),
        ("gemv_f32", "vecmat", capi.MV_F32_PLUS_TIMES, None, (N_MAT, N_MAT), mat_bytes),
        ("minplus_gevm_f32", "matvec", capi.MV_F32_MIN_PLUS, None, (N_MAT, N_MAT), mat_bytes),
    ]


def kernel_of(kind, op):
    from paper_2603_18695_b200 import capi
    if kind == "mapreduce":
        return "mapreduce_kernel"
    if kind == "scan":
        # 2^28-element scans: the lagged kernel for 16-byte carries, the
        # single-pass one otherwise (scan.cuh lag_scan_type_ok)
        return "scan_lag_kernel" if op in (capi.AFFINE_F32, capi.MAT2_U32) else "scan_smem_kernel"
    if kind == "matvec":
        return "gevm_cols_kernel"
    return "gemv_kernel"


# ---------------------------------------------------------------------------
# reference CPU arm (the reference VM compiled from /root/reference)

CPU_N = 1 << 23       # scans / mapreduces of the CPU sample (~0.2 s each on the reference VM)
CPU_MAT = 2048        # matrices of the CPU sample
CPU_C1 = 1 << 20      # BASELINE C1: inclusive f32 scan, "the reference CPU oracle run"


def cpu_sample_specs():
    from oracle import oracle as orc  # noqa: F401
    return [
        ("mapreduce_f32_sumsq", "mapreduce", 1, None, CPU_N),
        ("mapreduce_i32_max", "mapreduce", 6, None, CPU_N),
        ("scan_f32_sum_excl", "scan", 0, False, CPU_N),
        ("scan_affine_f32", "scan", 10, True, CPU_N),
        ("scan_argmax_f32i32", "scan", 11, True, CPU_N),
        ("gevm_f32", "matvec", 32, None, CPU_MAT),
        ("gemv_f32", "vecmat", 32, None, CPU_MAT),
        ("minplus_gevm_f32", "matvec", 33, None, CPU_MAT),
    ]


def cpu_composite(reps: int = 7, with_c1: bool = True) -> dict:
    """The reference's own CPU path (reference VM, Threads backend, timer =
    LaunchReport::wall_seconds) on a bounded sample of the
    composite (~10 s): every primitive at 2^23 elements / 2048^2, `reps` runs
    each; per primitive the median and minimum.  Also BASELINE C1 itself (the
    inclusive f32 scan at 2^20), reported beside, not in the value."""
    import numpy as np

    from oracle import oracle as orc
    kind_of = "reference" if orc.ref_available() else "port"
    per = {}
    tot_bytes = 0
    tot_med = 0.0
    specs = cpu_sample_specs() + ([("C1_scan_f32_sum_incl_2^20", "scan", 0, True, CPU_C1)] if with_c1 else [])
    for name, kind, op, incl, n in specs:
        ts = orc.t_dtype(op).itemsize
        ss = orc.s_dtype(op).itemsize
        if kind in ("matvec", "vecmat"):
            A = orc.fill(op, n * n, 0x5EED0C04)
            x = orc.fill(op, n, 0x5EED0C14)
            byts = n * n * ts + n * ts + n * ss
        else:
            x = orc.fill(op, n, 0x5EED0C01 + op)
            byts = n * ts + (n * ss if kind == "scan" else 0)
        times = []
        for _ in range(reps):
            t0 = time.perf_counter()
            if kind_of == "reference":
                if kind == "mapreduce":
                    _, w = orc.ref_mapreduce(op, x, backend=orc.THREADS)
                elif kind == "scan":
                    _, w = orc.ref_scan(op, incl, x, backend=orc.THREADS)
                elif kind == "matvec":
                    _, w = orc.ref_matvec(op, A, n, n, x, backend=orc.THREADS)
                else:
                    _, w = orc.ref_vecmat(op, A, n, n, x, backend=orc.THREADS)
            else:
                if kind == "mapreduce":
                    orc.mapreduce(op, x)
                elif kind == "scan":
                    orc.scan(op, incl, x)
                elif kind == "matvec":
                    orc.matvec(op, A, n, n, x)
                else:
                    orc.vecmat(op, A, n, n, x)
                w = time.perf_counter() - t0
            times.append(w)
        times.sort()
        med = times[len(times) // 2]
        per[name] = {"gbs": byts / med / 1e9, "median_s": med, "min_s": times[0], "runs": reps,
                     "bytes": byts, "n": n if kind not in ("matvec", "vecmat") else f"{n}x{n}"}
        if name.startswith("C1_"):
            per[name]["note"] = "BASELINE C1, reported beside the composite (not in value)"
            continue
        tot_bytes += byts
        tot_med += med
    if with_c1 and kind_of == "reference":
        # the reference's deterministic single-core backend (Backend::Simulator,
        # SURVEY.md §8(d)) on C1 as well: wall clock around the call
        x = orc.fill(0, CPU_C1, 0x5EED0C01)
        ts = []
        for _ in range(5):
            t0 = time.perf_counter()
            orc.ref_scan(0, True, x, backend=orc.SIM)
            ts.append(time.perf_counter() - t0)
        ts.sort()
        per["C1_scan_f32_sum_incl_2^20_simulator"] = {
            "gbs": CPU_C1 * 8 / ts[2] / 1e9, "median_s": ts[2], "min_s": ts[0], "runs": 5, "bytes": CPU_C1 * 8,
            "n": CPU_C1, "note": "reference VM Backend::Simulator (1 core, deterministic schedule); beside, not in value"}
    nproc = os.cpu_count() or 1
    workers = min(max(nproc, 2), 16)
    return {"value": tot_bytes / tot_med / 1e9, "unit": "GB/s",
            "cores": workers if kind_of == "reference" else 1, "kind": kind_of,
            "sample": f"the step's 8 primitives at 2^23 elements (scans, mapreduces) / 2048x2048 (matrices), "
                      f"{reps} runs each, median per primitive; reference VM Threads backend with "
                      f"clamp(hardware_concurrency,2,16) = {workers} workers (machine.cpp:1080-1084) on "
                      f"{nproc} host cores; timer LaunchReport::wall_seconds",
            "nproc": nproc, "workers": workers, "per_primitive": per}


def reference_arm(args, rank: int, world: int) -> None:
    if rank != 0:
        return
    t0 = time.perf_counter()
    for _ in range(args.warmup):
        cpu_composite(reps=1, with_c1=False)
    runs = [cpu_composite(reps=1, with_c1=False) for _ in range(args.steps)]
    wall = time.perf_counter() - t0
    vals = sorted(r["value"] for r in runs)
    value = vals[len(vals) // 2]
    last = runs[-1]
    byts = sum(v["bytes"] for v in last["per_primitive"].values())
    line = {
        "metric": METRIC, "impl": "reference", "value": value, "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * byts / (value * 1e9),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32+i32+struct",
        "data": "synthetic",
        "config": {"workload": "composite step (C2 mapreduces, C5/C3 scans, C4 matrices) on a bounded CPU "
                               "sample: scans and mapreduces at 2^23, matrices 2048x2048",
                   "wall_s": wall},
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": last["cores"], "kind": last["kind"],
                         "sample": last["sample"], "per_primitive": last["per_primitive"]},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# B200 arm


def forge_arm(args, rank: int, world: int, local_rank: int) -> None:
    import torch

    from paper_2603_18695_b200 import capi, dev, sharded
    from paper_2603_18695_b200.forge import op_info

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
        assert dist.get_world_size() == args.gpus, (dist.get_world_size(), args.gpus)
    stream = torch.cuda.current_stream()
    specs = component_specs()

    def max_over_ranks(v: float) -> float:
        if not dist:
            return v
        t = torch.tensor([v], device="cuda" if dist.get_backend() == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- inputs (global index = rank * n_local + i: the concatenation is the global array)
    bufs, outs = {}, {}
    be = sharded.DeviceBackend()
    for ci, (name, kind, op, incl, n, _) in enumerate(specs):
        seed = 0x5EED0010 + ci
        if kind in ("mapreduce", "scan"):
            x = dev.empty(op, n)
            dev.fill_synthetic(op, x, n, seed, index_base=rank * n)
            bufs[name] = x
            if kind == "scan":
                outs[name] = dev.empty(op, n, "S")
        else:
            rows, cols = n
            if "A" not in bufs:  # one 16384^2 block per rank serves all three matrix products
                A = dev.empty(op, rows * cols)
                dev.fill_synthetic(op, A, rows * cols, 0x5EED0C04, index_base=rank * rows * cols)
                bufs["A"] = A
            xl = rows if kind == "matvec" else cols
            x = dev.empty(op, xl)
            dev.fill_synthetic(op, x, xl, seed)
            bufs[name] = x
            outs[name] = dev.empty(op, cols if kind == "matvec" else rows, "S")

    def run_component(name, kind, op, incl, n):
        if kind == "mapreduce":
            return sharded.sharded_mapreduce(op, bufs[name], n, backend=be)
        if kind == "scan":
            return sharded.sharded_scan(op, incl, bufs[name], outs[name], n, backend=be)
        rows, cols = n
        if kind == "matvec":  # this rank's column block of the global rows x (cols*world) matrix
            return sharded.sharded_matvec(op, bufs["A"], rows, cols * world, bufs[name], outs[name], backend=be)
        return sharded.sharded_vecmat(op, bufs["A"], rows * world, cols, bufs[name], outs[name], backend=be)

    ev = []  # per step: [event before component 0, after 0, after 1, ...]

    def step(record: bool):
        if record:
            es = [torch.cuda.Event(enable_timing=True) for _ in range(len(specs) + 1)]
            es[0].record(stream)
        for ci, (name, kind, op, incl, n, _) in enumerate(specs):
            run_component(name, kind, op, incl, n)
            if record:
                es[ci + 1].record(stream)
        if record:
            ev.append(es)

    for _ in range(args.warmup):
        step(False)
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
            step(True)
        t1.record(stream)
        # steps are queued: sample while the GPU works through them (an NVML
        # query takes milliseconds — never between enqueues)
        sampler.sample_now()
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
    ms = max_over_ranks(t0.elapsed_time(t1))
    bytes_step = sum(b for *_, b in specs)
    value = world * bytes_step * args.steps / (ms * 1e-3) / 1e9
    elems_step = sum((n if isinstance(n, int) else n[0] * n[1]) for _, _, _, _, n, _ in specs)

    components = {}
    for ci, (name, kind, op, incl, n, byts) in enumerate(specs):
        cms = sum(es[ci].elapsed_time(es[ci + 1]) for es in ev) / len(ev)
        cms = max_over_ranks(cms)
        components[name] = {"ms_per_step": round(cms, 4), "bytes_per_gpu": byts,
                            "gbs_job": round(world * byts / (cms * 1e-3) / 1e9, 1),
                            "share_of_step": round(cms / (ms / args.steps), 4)}

    # ---- roofline: each kernel alone (CUDA events on its stream), N = 1 semantics per rank
    peaks = measured_peaks()
    traffic = traffic_table()
    ws_r = {"mapreduce": dev.Workspace(), "scan": dev.Workspace(), "matvec": dev.Workspace(),
            "vecmat": dev.Workspace()}
    o16 = torch.empty(16, dtype=torch.uint8, device="cuda")

    def kernel_call(name, kind, op, incl, n):
        if kind == "mapreduce":
            dev.mapreduce(op, bufs[name], n, o16, ws_r[kind], stream=stream)
        elif kind == "scan":
            dev.scan(op, incl, bufs[name], outs[name], n, ws_r[kind], stream=stream)
        elif kind == "matvec":
            dev.matvec(op, bufs["A"], n[0], n[1], bufs[name], outs[name], ws_r[kind], stream=stream)
        else:
            dev.vecmat(op, bufs["A"], n[0], n[1], bufs[name], outs[name], ws_r[kind], stream=stream)

    rooflines = {}
    for name, kind, op, incl, n, byts in specs:
        kernel_call(name, kind, op, incl, n)
        pairs = []
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            kernel_call(name, kind, op, incl, n)
            b.record(stream)
            pairs.append((a, b))
        torch.cuda.synchronize()
        kms = sorted(a.elapsed_time(b) for a, b in pairs)
        kavg = sum(kms) / len(kms)
        ach = byts / (kavg * 1e-3) / 1e9
        rooflines[name] = {"bound": "hbm", "achieved": round(ach, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
                           "frac": round(ach / peaks["hbm_gbs"], 4), "frac_of_nominal_8tbs": round(ach / 8000, 4),
                           "kernel": kernel_of(kind, op), "algorithmic_bytes_per_launch": byts,
                           "avg_launch_ms": round(kavg, 5), "traffic": traffic.get(name)}
    dominant = max(components, key=lambda k: components[k]["ms_per_step"])
    roofline = dict(rooflines[dominant])
    roofline.update({"component": dominant, "peak_source": peaks["source"],
                     "peak_note": "MEASURED_PEAKS hbm_gbs is a read+write copy (torch copy_); a read-only "
                                  "stream can exceed it (frac > 1)"})

    launches_per_step = 0
    for name, kind, op, incl, n, _ in specs:
        if kind == "mapreduce":
            launches_per_step += 1 if world == 1 else 2      # mapreduce (+ rank-order fold)
        elif kind == "scan":
            launches_per_step += 1 if world == 1 else 3      # scan (+ ordered shard reduce, carry fold)
        else:
            launches_per_step += 1

    line = {
        "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32+i32+struct", "data": "synthetic",
        "config": {"workload": "composite step of BASELINE configs per GPU: C2 mapreduce f32 sum-of-squares + "
                               "i32 max (2^30 each), C5-op exclusive f32 scan + C3 affine and argmax scans "
                               "(2^28 each), C4 gevm + gemv + min-plus gevm (16384^2); global problems sharded "
                               "across ranks (weak scaling)",
                   "bytes_per_gpu_per_step": bytes_step, "elems_per_gpu_per_step": elems_step,
                   "l2": "inputs >> 126 MB L2 (21 GiB touched per GPU per step); no flush needed",
                   "parallelism": f"shard{world}"},
        "elems_per_s": world * elems_step * args.steps / (ms * 1e-3),
        "components": components,
        "roofline": roofline,
        "rooflines": rooflines,
        "gpu_launches": args.steps * launches_per_step,
        "clocks": sampler.summary(),
    }
    # free the composite's inputs before the C5 leg (64 GiB at N = 1)
    del bufs, outs
    torch.cuda.empty_cache()
    if not args.no_c5:
        line["c5"] = c5_leg(args, rank, world, dist, max_over_ranks)
        torch.cuda.empty_cache()
    if not args.no_e2e:
        line["e2e"] = e2e_leg(args, rank, world, dist, max_over_ranks)
        torch.cuda.empty_cache()
    if rank == 0 and world == 1 and not args.no_breakdown:
        line["context"] = context_breakdown(peaks)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_composite()
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def c5_leg(args, rank, world, dist, max_over_ranks) -> dict:
    """BASELINE C5: n = 2^33 f32 GLOBAL, contiguous shards of 2^33/N per GPU
    (strong scaling): sharded exclusive scan and sharded mapreduce (sum),
    device-timed, max over ranks; whole-job algorithmic GB/s."""
    import torch

    from paper_2603_18695_b200 import capi, dev, sharded
    n_local = N_C5 // world
    op = capi.F32_SUM
    x = dev.empty(op, n_local)
    dev.fill_synthetic(op, x, n_local, 0x5EED0C05, index_base=rank * n_local)
    y = dev.empty(op, n_local, "S")
    be = sharded.DeviceBackend()
    s = torch.cuda.current_stream()
    out = {}
    for name, fn, byts in (("exclusive_scan_f32", lambda: sharded.sharded_scan(op, False, x, y, n_local, backend=be),
                            N_C5 * 8),
                           ("mapreduce_f32_sum", lambda: sharded.sharded_mapreduce(op, x, n_local, backend=be),
                            N_C5 * 4)):
        fn()
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        reps = 3
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(reps):
            fn()
        b.record(s)
        torch.cuda.synchronize()
        ms = max_over_ranks(a.elapsed_time(b) / reps)
        out[name] = {"gbs": round(byts / (ms * 1e-3) / 1e9, 1), "ms": round(ms, 4),
                     "elems_per_s": float(f"{N_C5 / (ms * 1e-3):.4g}"), "algorithmic_bytes": byts}
    out["config"] = {"n_global": N_C5, "n_per_gpu": n_local, "scaling": "strong",
                     "scan": "reduce-then-scan (ordered shard reduce, all-gather of totals, rank-order fold, "
                             "carry-seeded single-pass scan): 3n/N bytes per GPU at N > 1",
                     "exchange": (f"{dist.get_backend()} all-gather of sizeof(S) per rank" if world > 1 else "none")}
    del x, y
    return out


def e2e_leg(args, rank, world, dist, max_over_ranks) -> dict:
    """The composite through the public API with HOST buffers: every step, each
    input goes host (pinned) -> device (forge_write_bytes through the C-ABI
    Machine at N = 1; torch copy at N > 1), the primitives run (C-ABI Machine
    calls at N = 1: forge_mapreduce returns its value to the host; sharded.py at
    N > 1), and every result comes back to the host (the scans' full outputs,
    the matrix outputs, the mapreduce values).  Wall clock around the steps,
    barriers on both sides, the slowest rank's time."""
    import numpy as np
    import torch

    from paper_2603_18695_b200 import dev, sharded
    from paper_2603_18695_b200 import forge as F
    specs = component_specs()
    host_in, host_out = {}, {}
    for ci, (name, kind, op, incl, n, _) in enumerate(specs):
        seed = 0x5EED0010 + ci
        if kind in ("mapreduce", "scan"):
            t = dev.empty(op, n)
            dev.fill_synthetic(op, t, n, seed, index_base=rank * n)
        else:
            rows, cols = n
            if "A" not in host_in:
                A = dev.empty(op, rows * cols)
                dev.fill_synthetic(op, A, rows * cols, 0x5EED0C04, index_base=rank * rows * cols)
                host_in["A"] = torch.empty(A.numel(), dtype=torch.uint8, pin_memory=True)
                host_in["A"].copy_(A)
                del A
            xl = rows if kind == "matvec" else cols
            t = dev.empty(op, xl)
            dev.fill_synthetic(op, t, xl, seed)
        h = torch.empty(t.numel(), dtype=torch.uint8, pin_memory=True)
        h.copy_(t)
        host_in[name] = h
        del t
        if kind == "scan":
            host_out[name] = torch.empty(n * op_size(op, "S"), dtype=torch.uint8, pin_memory=True)
        elif kind in ("matvec", "vecmat"):
            host_out[name] = torch.empty((n[1] if kind == "matvec" else n[0]) * op_size(op, "S"), dtype=torch.uint8,
                                         pin_memory=True)
    torch.cuda.empty_cache()
    h2d = sum(h.numel() for h in host_in.values())
    d2h = sum(h.numel() for h in host_out.values()) + sum(op_size(op, "S") for _, k, op, *_ in specs
                                                           if k == "mapreduce")
    byts = sum(b for *_, b in specs)

    if world == 1:
        m = F.Machine(torch.cuda.current_device())
        mb, ws = {}, {}
        for name, kind, op, incl, n, _ in specs:
            if kind in ("mapreduce", "scan"):
                mb[name] = F.create_buffer(m, op, n)
                if kind == "scan":
                    mb[name + ".out"] = F.create_buffer(m, op, n, which="S")
                    ws[name] = F.make_scan_workspace(m, op, n)
                else:
                    ws[name] = F.make_mapreduce_workspace(m, op)
            else:
                rows, cols = n
                if "A" not in mb:
                    mb["A"] = F.create_buffer(m, op, rows * cols)
                mb[name] = F.create_buffer(m, op, rows if kind == "matvec" else cols)
                mb[name + ".out"] = F.create_buffer(m, op, cols if kind == "matvec" else rows, which="S")
                ws[name] = F.make_mat_workspace(m, op, rows, cols)
        results = {}

        def step():
            m.write_ptr(mb["A"], host_in["A"].data_ptr(), host_in["A"].numel())
            for name, kind, op, incl, n, _ in specs:
                m.write_ptr(mb[name], host_in[name].data_ptr(), host_in[name].numel())
                if kind == "mapreduce":
                    results[name], _ = F.mapreduce(m, F.make_semiring(op), F.make_view(m, mb[name]), ws[name])
                elif kind == "scan":
                    F.scan(m, F.make_semiring(op), F.make_view(m, mb[name]), F.make_view(m, mb[name + ".out"]), incl,
                           ws[name])
                    m.read_ptr(mb[name + ".out"], host_out[name].data_ptr(), host_out[name].numel())
                else:
                    rows, cols = n
                    fn = F.matvec if kind == "matvec" else F.vecmat
                    fn(m, F.make_semiring(op), F.make_view(m, mb["A"]), rows, cols, F.make_view(m, mb[name]),
                       F.make_view(m, mb[name + ".out"]), ws[name])
                    m.read_ptr(mb[name + ".out"], host_out[name].data_ptr(), host_out[name].numel())
        path = ("C-ABI Machine: forge_write_bytes (pinned host -> HBM) for every input, forge_mapreduce (value "
                "to the host) / forge_scan / forge_matvec / forge_vecmat, forge_read_bytes of every output")
    else:
        dbufs = {k: torch.empty(h.numel(), dtype=torch.uint8, device="cuda") for k, h in host_in.items()}
        douts = {k: torch.empty(h.numel(), dtype=torch.uint8, device="cuda") for k, h in host_out.items()}
        be = sharded.DeviceBackend()

        def step():
            for k, h in host_in.items():
                dbufs[k].copy_(h, non_blocking=True)
            vals = []
            for name, kind, op, incl, n, _ in specs:
                if kind == "mapreduce":
                    vals.append(sharded.sharded_mapreduce(op, dbufs[name], n, backend=be))
                elif kind == "scan":
                    sharded.sharded_scan(op, incl, dbufs[name], douts[name], n, backend=be)
                elif kind == "matvec":
                    sharded.sharded_matvec(op, dbufs["A"], n[0], n[1] * world, dbufs[name], douts[name], backend=be)
                else:
                    sharded.sharded_vecmat(op, dbufs["A"], n[0] * world, n[1], dbufs[name], douts[name], backend=be)
            for k, h in host_out.items():
                h.copy_(douts[k], non_blocking=True)
            for v in vals:
                v.cpu()
            torch.cuda.synchronize()
        path = ("sharded.py on device buffers: pinned host -> HBM copy of every input, sharded_mapreduce / "
                "sharded_scan / sharded_matvec / sharded_vecmat (NCCL exchanges), HBM -> pinned host copy of "
                "every output")

    def timed(fn, k=3):
        fn()
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(k):
            fn()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if dist:
            dist.barrier()
        return max_over_ranks(dt), k

    sync_dt, k = timed(step)
    sync_path = path
    if world == 1:
        m.close()
        del mb, ws

    # ---- the same step pipelined over full-duplex PCIe: component i's inputs go
    # up on an H2D stream while component i-1 computes and component i-2's
    # outputs come down on a D2H stream (device-pointer C-ABI layer on the
    # compute stream; every input and output still crosses PCIe every step)
    be = sharded.DeviceBackend()
    s_up, s_comp, s_down = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    din = {k_: torch.empty(h.numel(), dtype=torch.uint8, device="cuda") for k_, h in host_in.items()}
    dout = {k_: torch.empty(h.numel(), dtype=torch.uint8, device="cuda") for k_, h in host_out.items()}
    mr_host = {name: torch.empty(16, dtype=torch.uint8, pin_memory=True) for name, kind, *_ in specs
               if kind == "mapreduce"}
    ev = lambda: torch.cuda.Event()  # noqa: E731
    prev_done = {}   # component -> event: its compute finished (its inputs may be overwritten)
    prev_down = {}   # component -> event: its outputs were read back (its outputs may be overwritten)

    def step_pipelined():
        a_up = None
        for name, kind, op, incl, n, _ in specs:
            keys = [name] + (["A"] if kind in ("matvec", "vecmat") and a_up is None else [])
            with torch.cuda.stream(s_up):
                for key in keys:
                    if key in prev_done:
                        s_up.wait_event(prev_done[key])
                    din[key].copy_(host_in[key], non_blocking=True)
                up = ev()
                up.record(s_up)
                if "A" in keys:
                    a_up = up
            with torch.cuda.stream(s_comp):
                s_comp.wait_event(up)
                if kind in ("matvec", "vecmat"):
                    s_comp.wait_event(a_up)
                if name in prev_down:
                    s_comp.wait_event(prev_down[name])
                if kind == "mapreduce":
                    val = sharded.sharded_mapreduce(op, din[name], n, backend=be)
                elif kind == "scan":
                    sharded.sharded_scan(op, incl, din[name], dout[name], n, backend=be)
                elif kind == "matvec":
                    sharded.sharded_matvec(op, din["A"], n[0], n[1] * world, din[name], dout[name], backend=be)
                else:
                    sharded.sharded_vecmat(op, din["A"], n[0] * world, n[1], din[name], dout[name], backend=be)
                done = ev()
                done.record(s_comp)
                prev_done[name] = done
                if kind in ("matvec", "vecmat"):
                    prev_done["A"] = done
            with torch.cuda.stream(s_down):
                s_down.wait_event(done)
                if kind == "mapreduce":
                    val.record_stream(s_down)
                    mr_host[name][: val.numel()].copy_(val, non_blocking=True)
                else:
                    host_out[name].copy_(dout[name], non_blocking=True)
                dn = ev()
                dn.record(s_down)
                prev_down[name] = dn
        s_down.synchronize()  # every result on the host

    pipe_dt, k = timed(step_pipelined)
    del din, dout
    torch.cuda.empty_cache()
    pipe_path = ("device-pointer C-ABI (forge_dev_*, through sharded.py at every N) on a compute stream; pinned "
                 "host -> HBM copies of every input on an H2D stream and HBM -> pinned host copies of every output "
                 "on a D2H stream, pipelined across the step's components (PCIe is full duplex)")
    return {"value": world * byts * k / pipe_dt / 1e9, "unit": "GB/s", "h2d_bytes_per_step": world * h2d,
            "d2h_bytes_per_step": world * d2h, "path": pipe_path, "steps": k, "ms_per_step": 1e3 * pipe_dt / k,
            "unpipelined": {"value": world * byts * k / sync_dt / 1e9, "ms_per_step": 1e3 * sync_dt / k,
                            "path": sync_path}}


def op_size(op, which="T"):
    from paper_2603_18695_b200.forge import op_info
    return op_info(op)["t_size" if which == "T" else "s_size"]


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


def context_breakdown(peaks) -> dict:
    """Context numbers outside the timed region (median of 5 event pairs):
    vcopy calibration, the C1 launch-bound scan (direct and CUDA graph), the
    UnitFloat8 promotion, min-plus gemv, i32 scan."""
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
    nb = 2 * GIB
    a = torch.empty(nb, dtype=torch.uint8, device="cuda")
    b = torch.empty(nb, dtype=torch.uint8, device="cuda")
    rec("vcopy_2GiB", 2 * nb, _time_dev(lambda: dev.copy(a, b, nb)))
    rec("torch_copy_2GiB", 2 * nb, _time_dev(lambda: b.copy_(a)))
    del a, b
    n = 1 << 28
    src = dev.empty(capi.I32_SUM, n)
    dev.fill_synthetic(capi.I32_SUM, src, n, 3)
    dst = dev.empty(capi.I32_SUM, n, "S")
    rec("scan_i32_sum_2^28", n * 8, _time_dev(lambda: dev.scan(capi.I32_SUM, True, src, dst, n, ws)), elems=n)
    del src, dst
    n1 = 1 << 20
    src = dev.empty(capi.F32_SUM, n1)
    dev.fill_synthetic(capi.F32_SUM, src, n1, 1)
    dst = dev.empty(capi.F32_SUM, n1, "S")
    rec("scan_f32_sum_2^20_C1", n1 * 8, _time_dev(lambda: dev.scan(capi.F32_SUM, True, src, dst, n1, ws), 20),
        elems=n1, note="8 MiB, L2-resident: one call per event pair, host launch latency included")

    def c1_calls():
        for _ in range(100):
            dev.scan(capi.F32_SUM, True, src, dst, n1, ws)
    rec("scan_f32_sum_2^20_C1_back_to_back", n1 * 8, _time_dev(c1_calls, 5) / 100, elems=n1,
        note="100 calls through the Python device-pointer layer between one event pair; per-call time "
             "(max of the host call cost and the kernel)")
    try:
        gstream = torch.cuda.Stream()
        gstream.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(gstream):
            for _ in range(3):
                dev.scan(capi.F32_SUM, True, src, dst, n1, ws, stream=gstream)
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
    nn = 16384
    A = dev.empty(capi.MV_F32_MIN_PLUS, nn * nn)
    dev.fill_synthetic(capi.MV_F32_MIN_PLUS, A, nn * nn, 5)
    x = dev.empty(capi.MV_F32_MIN_PLUS, nn)
    dev.fill_synthetic(capi.MV_F32_MIN_PLUS, x, nn, 6)
    y = dev.empty(capi.MV_F32_MIN_PLUS, nn, "S")
    rec("minplus_gemv_f32_16384^2", nn * nn * 4 + 2 * nn * 4,
        _time_dev(lambda: dev.vecmat(capi.MV_F32_MIN_PLUS, A, nn, nn, x, y, ws)), elems=nn * nn)
    del A
    src = dev.empty(capi.UF8_F32_SUM, N_MR)
    dev.fill_synthetic(capi.UF8_F32_SUM, src, N_MR, 7)
    outb = torch.zeros(16, dtype=torch.uint8, device="cuda")
    rec("mapreduce_uf8_f32_2^30", N_MR, _time_dev(lambda: dev.mapreduce(capi.UF8_F32_SUM, src, N_MR, outb, ws)),
        elems=N_MR)
    del src
    torch.cuda.empty_cache()
    return out


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["forge", "reference"], default="forge")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-c5", action="store_true")
    ap.add_argument("--no-breakdown", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # one process per GPU: re-launch under torch.distributed.run
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={_free_port()}", str(Path(__file__).resolve())] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}")
    if args.impl == "reference":
        reference_arm(args, rank, world)
        return
    forge_arm(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
