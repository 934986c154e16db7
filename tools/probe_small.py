"""Scan time at small / medium n, CUDA-graph replays (development)."""
import json
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2603_18695_b200 import capi, dev  # noqa: E402

op = capi.F32_SUM
out = {}
for lg in (18, 20, 21, 22, 23, 24, 25, 26, 27):
    n = 1 << lg
    src = dev.empty(op, n)
    dev.fill_synthetic(op, src, n, 1)
    dst = dev.empty(op, n, "S")
    ws = dev.Workspace()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            dev.scan(op, True, src, dst, n, ws)
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(10):
            dev.scan(op, True, src, dst, n, ws)
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    us = a.elapsed_time(b) / 50 * 1e3
    out[f"2^{lg}"] = {"us": round(us, 2), "gbs": round(n * 8 / us / 1e3, 1)}
print(json.dumps(out))
