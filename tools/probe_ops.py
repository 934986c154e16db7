"""Scan GB/s of every lag-eligible menu op at 2^28 (2^27 for 16-byte elements) (development).
FORGE_LIB=dev FORGE_SCAN_LAG=0 selects the single-pass kernel."""
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


ws = dev.Workspace()
out = {}
for name in ("F32_SUM", "F32_SUMSQ", "F32_MAX", "F64_SUM", "I32_SUM", "I32_MAX", "U32_SUM", "I64_SUM",
             "AFFINE_F32", "ARGMAX_F32I32", "MAT2_U32", "LSE_F32", "QUAT_F32"):
    op = getattr(capi, name, None)
    if op is None:
        continue
    inf = op_info(op)
    n = 1 << 28 if inf["t_size"] <= 8 else 1 << 27
    src = dev.empty(op, n); dev.fill_synthetic(op, src, n, 3); dst = dev.empty(op, n, "S")
    try:
        ms = t(lambda: dev.scan(op, True, src, dst, n, ws))
        out[name] = round(n * (inf["t_size"] + inf["s_size"]) / ms / 1e6, 1)
    except Exception as e:
        out[name] = str(e)[:60]
    del src, dst
print(json.dumps({"lag": os.environ.get("FORGE_SCAN_LAG", "default"), "gbs": out}))
