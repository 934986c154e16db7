"""Lagged scan with / without the row-prefix ring (forge_set_scan_ring_bypass), 2^28 (development)."""
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
    x = sorted(a.elapsed_time(b) for a, b in ev); return x[len(x) // 2]


lib = capi.load()
ws = dev.Workspace()
out = {}
for name, op in (("i64", capi.I64_SUM), ("f64", capi.F64_SUM), ("argmax", capi.ARGMAX_F32I32),
                 ("f32", capi.F32_SUM), ("affine", capi.AFFINE_F32), ("mat2", capi.MAT2_U32)):
    inf = op_info(op)
    n = 1 << 28 if inf["t_size"] <= 8 else 1 << 27
    src = dev.empty(op, n); dev.fill_synthetic(op, src, n, 3); dst = dev.empty(op, n, "S")
    r = {}
    for byp in (0, 1, 0):
        lib.forge_set_scan_ring_bypass(byp)
        ms = t(lambda: dev.scan(op, True, src, dst, n, ws))
        r[f"bypass{byp}"] = round(n * (inf["t_size"] + inf["s_size"]) / ms / 1e6, 1)
    lib.forge_set_scan_ring_bypass(0)
    out[name] = r
    del src, dst
print(json.dumps(out))
