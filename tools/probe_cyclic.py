"""Cyclic sharded scan throughput on one GPU (development): G = 1 and emulated
G = 2 / 4 groups, 2^28 f32 inclusive, chunk = tpc tiles."""
import json
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2603_18695_b200 import capi, dev, group  # noqa: E402

op, n = capi.F32_SUM, 1 << 28
out = {}
for G in (1, 2, 4):
    q = group.cyclic_quantum(op)
    for tpc in sorted({16, max(1, 148 // G)}):
        if tpc * G > 148 and G > 1:
            continue
        chunk = tpc * q
        with group.Group([0] * G) as g:
            src, dst = [], []
            for r in range(G):
                ln = group.cyclic_local_n(n, chunk, r, G)
                s = dev.empty(op, ln)
                dev.fill_synthetic(op, s, ln, 3)
                src.append(s)
                dst.append(dev.empty(op, ln, "S"))
            for _ in range(3):
                g.scan_cyclic(op, True, src, dst, n, chunk)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(10):
                g.scan_cyclic(op, True, src, dst, n, chunk)
            b.record()
            torch.cuda.synchronize()
            ms = a.elapsed_time(b) / 10
            out[f"G{G}_tpc{tpc}"] = round(n * 8 / ms / 1e6, 1)
            del src, dst
            torch.cuda.empty_cache()
print(json.dumps({"cyclic_scan_f32_2^28_gbs": out}))
