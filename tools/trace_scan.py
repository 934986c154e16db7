"""Per-tile phase timing of the smem scan kernel (development tool; needs the
DEV library: make -C paper_2603_18695_b200/csrc DEV=1).
    FORGE_LIB=dev python tools/trace_scan.py [op] [log2n]"""
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
host = buf.cpu().numpy().view(np.uint64)
raw = host.reshape(-1, 8).astype(np.int64)
raw = raw[raw[:, 0] > 0]
t0 = raw[:, 0].min()
ph = raw[:, :5] - t0
d = {"tiles": len(raw), "span_us": float((ph[:, 4].max()) / 1e3)}
for i, name in enumerate(["claim->landed", "landed->pass1", "pass1->prefix", "prefix->end"]):
    x = (ph[:, i + 1] - ph[:, i]) / 1e3
    d[name] = {"mean_us": round(float(x.mean()), 3), "p50": round(float(np.median(x)), 3),
               "p90": round(float(np.percentile(x, 90)), 3), "max": round(float(x.max()), 3)}
sc = (raw[:, 0] - raw[:, 7]) / 1e3
d["start->claim"] = {"mean_us": round(float(sc.mean()), 3), "p50": round(float(np.median(sc)), 3)}
life = (ph[:, 4] - (raw[:, 7] - t0)) / 1e3
d["lifetime_us"] = {"mean": round(float(life.mean()), 3), "p50": round(float(np.median(life)), 3)}
mid = ph[:, 4].max() / 2
d["alive_at_mid"] = int(((ph[:, 0] <= mid) & (ph[:, 4] >= mid)).sum())
d["distinct_sms"] = int(len(np.unique(raw[:, 5])))
st = np.sort(ph[:, 0])
d["claims_per_us"] = float(len(st) / (st[-1] - st[0]) * 1e3)
rounds = raw[:, 6]
sel = rounds > 0
d["lookback_rounds_mean"] = float(rounds[sel].mean()) if sel.any() else 0.0
d["lookback_rounds_p90"] = float(np.percentile(rounds[sel], 90)) if sel.any() else 0.0
lb = (ph[:, 3] - ph[:, 2]) / 1e3
d["us_per_round"] = float((lb[sel] / np.maximum(rounds[sel], 1)).mean()) if sel.any() else 0.0
print(json.dumps(d))
