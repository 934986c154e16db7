"""Per-ticket phase timing of the lagged scan (development tool; DEV library).
    FORGE_LIB=dev python tools/trace_lag.py [op] [log2n]"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["FORGE_SCAN_TRACE"] = "1"
os.environ["FORGE_LIB"] = "dev"
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2603_18695_b200 import capi, dev  # noqa: E402

op = int(sys.argv[1]) if len(sys.argv) > 1 else capi.F32_SUM
n = 1 << (int(sys.argv[2]) if len(sys.argv) > 2 else 28)
ws = dev.Workspace()
src = dev.empty(op, n)
dev.fill_synthetic(op, src, n, 3)
dst = dev.empty(op, n, "S")
for _ in range(3):
    dev.scan(op, True, src, dst, n, ws)
torch.cuda.synchronize()
lib = capi.load()
ptr, words = C.c_void_p(), C.c_uint64()
lib.forge_dev_scan_trace(C.byref(ptr), C.byref(words))
buf = torch.empty(words.value * 8, dtype=torch.uint8, device="cuda")
lib.forge_dev_copy(ptr, C.c_void_p(buf.data_ptr()), C.c_uint64(words.value * 8), None)
raw = buf.cpu().numpy().view(np.uint64).reshape(-1, 8).astype(np.int64)
raw = raw[raw[:, 0] > 0]
t0 = raw[:, 0].min()


def span(a, b):
    sel = (raw[:, a] > 0) & (raw[:, b] > 0)
    x = (raw[sel, b] - raw[sel, a]) / 1e3
    return {"mean_us": round(float(x.mean()), 3), "p50": round(float(np.median(x)), 3), "count": int(sel.sum())}


end = np.where(raw[:, 7] > 0, raw[:, 7], np.where(raw[:, 3] > 0, raw[:, 3], raw[:, 1]))
d = {"tickets": len(raw), "span_us": round(float((end.max() - t0) / 1e3), 1),
     "start->claim": span(0, 1), "claim->A_landed": span(1, 2), "A_landed->A_published": span(2, 3),
     "claim->carry_ready": span(1, 4), "A_published->B_landed": span(3, 5), "carry_ready->B_landed": span(4, 5),
     "B_landed->store_issued": span(5, 6), "store_issued->end": span(6, 7),
     "lifetime_AB_us": span(0, 7)}
life = (end - raw[:, 0]) / 1e3
d["lifetime_all_mean_us"] = round(float(life.mean()), 3)
mid = (end.max() + t0) / 2
d["alive_at_mid"] = int(((raw[:, 0] <= mid) & (end >= mid)).sum())
d["ticket_ne_blockidx_frac"] = round(float((raw[:, 1] & 1).mean()), 4)
miss = (raw[:, 1] & 1) == 1
if miss.any() and (~miss).any():
    la = (raw[:, 2] - raw[:, 0]) / 1e3
    ok2 = raw[:, 2] > 0
    d["start->A_landed_ticket_eq_blockidx_us"] = round(float(la[ok2 & ~miss].mean()), 3)
    d["start->A_landed_ticket_ne_blockidx_us"] = round(float(la[ok2 & miss].mean()), 3)
print(json.dumps(d))
