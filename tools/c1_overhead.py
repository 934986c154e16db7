"""Per-call host cost of the C1 scan (2^20 f32, L2-resident) through the layers
(development tool): Python dev.scan, a prebuilt ctypes call, and the GPU time
alone (CUDA graph).  Wall-clock per call over 2000 back-to-back calls."""
import ctypes as C
import json
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2603_18695_b200 import capi, dev  # noqa: E402

n = 1 << 20
op = capi.F32_SUM
src = dev.empty(op, n)
dev.fill_synthetic(op, src, n, 1)
dst = dev.empty(op, n, "S")
ws = dev.Workspace()
out = {}


def wall(fn, k=2000):
    for _ in range(50):
        fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(k):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / k * 1e6


out["dev.scan_us"] = wall(lambda: dev.scan(op, True, src, dst, n, ws))
lib = capi.load()
w, wb = ws.for_(capi.PRIM_SCAN, op, n)
s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
args = (op, 1, src.data_ptr(), dst.data_ptr(), n, None, None, w, wb, s)
f = lib.forge_dev_scan
out["ctypes_prebuilt_us"] = wall(lambda: f(*args))
out["torch_current_stream_us"] = wall(lambda: torch.cuda.current_stream(), 20000)
plan = dev.ScanPlan(op, True, src, dst, n, ws) if hasattr(dev, "ScanPlan") else None
if plan:
    out["ScanPlan_us"] = wall(plan)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    for _ in range(20):
        dev.scan(op, True, src, dst, n, ws)
out["graph_gpu_us_per_scan"] = wall(lambda: g.replay(), 200) / 20
print(json.dumps({k: round(v, 2) for k, v in out.items()}))
