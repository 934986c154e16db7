#!/usr/bin/env python3
"""Quick kernel timing probe (development tool, not the bench contract).
usage: python tools/probe.py scan|mapreduce|matrix [--check]"""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2603_18695_b200 import capi, dev
from paper_2603_18695_b200.forge import op_info

def t(fn, reps=10):
    s = torch.cuda.current_stream(); fn(); torch.cuda.synchronize()
    ev = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s); fn(); b.record(s); ev.append((a, b))
    torch.cuda.synchronize()
    x = sorted(a.elapsed_time(b) for a, b in ev); return x[len(x)//2]

what = sys.argv[1] if len(sys.argv) > 1 else "scan"
check = "--check" in sys.argv
ws = dev.Workspace(); out = {}
if what == "scan":
    n = 1 << 28
    for name, op, incl in (("f32_incl", capi.F32_SUM, True), ("i32_incl", capi.I32_SUM, True),
                           ("affine", capi.AFFINE_F32, True), ("argmax", capi.ARGMAX_F32I32, True),
                           ("mat2", capi.MAT2_U32, True)):
        nn = n if op_info(op)["t_size"] <= 8 else n // 2
        src = dev.empty(op, nn); dev.fill_synthetic(op, src, nn, 3); dst = dev.empty(op, nn, "S")
        ms = t(lambda: dev.scan(op, incl, src, dst, nn, ws))
        inf = op_info(op); gbs = nn * (inf["t_size"] + inf["s_size"]) / ms / 1e6
        out[name] = round(gbs, 1)
        if check:
            from oracle import oracle as orc
            import numpy as np
            got = dst.cpu().numpy().view(orc.s_dtype(op))
            bad, worst = orc.check_scan_synthetic(op, incl, nn, 3, got, 1e-5)
            out[name + "_bad"] = bad
        del src, dst
print(json.dumps({"path": os.environ.get("FORGE_SCAN_PATH", "tile"), what: out}))
if what == "mapreduce":
    n = 1 << 30
    for name, op in (("f32_sumsq", capi.F32_SUMSQ), ("i32_max", capi.I32_MAX), ("uf8_f32_sum", capi.UF8_F32_SUM)):
        src = dev.empty(op, n); dev.fill_synthetic(op, src, n, 7)
        out_t = torch.zeros(16, dtype=torch.uint8, device="cuda")
        ms = t(lambda: dev.mapreduce(op, src, n, out_t, ws))
        out[name] = round(n * op_info(op)["t_size"] / ms / 1e6, 1)
        if check:
            from oracle import oracle as orc
            import numpy as np
            got = out_t.cpu().numpy().view(np.uint8)[: orc.s_dtype(op).itemsize].view(orc.s_dtype(op))
            want, ex, sc = orc.mapreduce_synthetic(op, n, 7)
            out[name + "_ok"] = bool(orc.within(op, got, ex, sc, 1e-5)[0]) if orc.ncomp(op) else bool(got[0] == want)
        del src
    print(json.dumps({"mapreduce": out}))
if what == "matrix":
    nn = 16384
    op = capi.MV_F32_PLUS_TIMES
    A = dev.empty(op, nn * nn); dev.fill_synthetic(op, A, nn * nn, 5)
    x = dev.empty(op, nn); dev.fill_synthetic(op, x, nn, 6)
    y = dev.empty(op, nn, "S")
    byts = nn * nn * 4 + 2 * nn * 4
    out["gevm"] = round(byts / t(lambda: dev.matvec(op, A, nn, nn, x, y, ws)) / 1e6, 1)
    out["gemv"] = round(byts / t(lambda: dev.vecmat(op, A, nn, nn, x, y, ws)) / 1e6, 1)
    o16 = torch.zeros(16, dtype=torch.uint8, device="cuda")
    out["mapreduce_1GiB"] = round(nn * nn * 4 / t(lambda: dev.mapreduce(capi.F32_SUMSQ, A, nn * nn, o16, ws)) / 1e6, 1)
    print(json.dumps({"matrix": out}))
if what == "copy":
    nb = 2 << 30
    a = torch.empty(nb, dtype=torch.uint8, device="cuda"); b = torch.empty(nb, dtype=torch.uint8, device="cuda")
    out["forge_copy"] = round(2 * nb / t(lambda: dev.copy(a, b, nb)) / 1e6, 1)
    out["torch_copy"] = round(2 * nb / t(lambda: b.copy_(a)) / 1e6, 1)
    print(json.dumps({"copy": out}))
if what == "c1":
    for n in (1 << 16, 1 << 18, 1 << 20, 1 << 22):
        op = capi.F32_SUM
        src = dev.empty(op, n); dev.fill_synthetic(op, src, n, 1); dst = dev.empty(op, n, "S")
        ms = t(lambda: dev.scan(op, True, src, dst, n, ws), 50)
        out[f"scan_f32_2^{n.bit_length()-1}_us"] = round(ms * 1e3, 2)
        if check:
            from oracle import oracle as orc
            got = dst.cpu().numpy().view(orc.s_dtype(op))
            out[f"bad_2^{n.bit_length()-1}"] = orc.check_scan_synthetic(op, True, n, 1, got, 1e-5)[0]
    print(json.dumps({"c1": out}))
if what == "c1g":
    n1 = 1 << 20
    op = capi.F32_SUM
    src = dev.empty(op, n1); dev.fill_synthetic(op, src, n1, 1); dst = dev.empty(op, n1, "S")
    g = torch.cuda.CUDAGraph()
    for _ in range(3): dev.scan(op, True, src, dst, n1, ws)
    torch.cuda.synchronize()
    with torch.cuda.graph(g):
        for _ in range(20): dev.scan(op, True, src, dst, n1, ws)
    out["graph_us_per_scan"] = round(t(lambda: g.replay(), 10) * 1e3 / 20, 2)
    out["single_us"] = round(t(lambda: dev.scan(op, True, src, dst, n1, ws), 50) * 1e3, 2)
    if check:
        from oracle import oracle as orc
        g.replay(); torch.cuda.synchronize()
        got = dst.cpu().numpy().view(orc.s_dtype(op))
        out["bad"] = orc.check_scan_synthetic(op, True, n1, 1, got, 1e-5)[0]
    print(json.dumps({"c1g": out}))
if what == "bigthen":
    def mx(tag):
        nn = 16384
        op = capi.MV_F32_PLUS_TIMES
        A = dev.empty(op, nn * nn); dev.fill_synthetic(op, A, nn * nn, 5)
        x = dev.empty(op, nn); dev.fill_synthetic(op, x, nn, 6)
        y = dev.empty(op, nn, "S")
        byts = nn * nn * 4 + 2 * nn * 4
        out[tag + "_gevm"] = round(byts / t(lambda: dev.matvec(op, A, nn, nn, x, y, ws)) / 1e6, 1)
        out[tag + "_gemv"] = round(byts / t(lambda: dev.vecmat(op, A, nn, nn, x, y, ws)) / 1e6, 1)
    mx("before")
    n5 = 1 << 33
    src = dev.empty(capi.F32_SUM, n5); dev.fill_synthetic(capi.F32_SUM, src, n5, 1)
    dst = dev.empty(capi.F32_SUM, n5, "S")
    dev.scan(capi.F32_SUM, False, src, dst, n5, ws); torch.cuda.synchronize()
    mx("during")
    del src, dst
    mx("after_del")
    torch.cuda.empty_cache()
    mx("after_empty")
    ws2 = dev.Workspace()
    ws = ws2
    mx("fresh_ws")
    print(json.dumps({"bigthen": out}))
if what == "ordered":
    for name, op in (("f32_sum", capi.F32_SUM), ("mat2", capi.MAT2_U32), ("affine", capi.AFFINE_F32)):
        n = (1 << 30) if op_info(op)["t_size"] <= 4 else (1 << 28)
        src = dev.empty(op, n); dev.fill_synthetic(op, src, n, 7)
        o = torch.zeros(32, dtype=torch.uint8, device="cuda")
        out[name] = round(n * op_info(op)["t_size"] / t(lambda: dev.reduce_ordered(op, src, n, o, ws)) / 1e6, 1)
        del src
    print(json.dumps({"ordered": out}))
