"""Per-tile phase timing of the smem scan kernel (development tool).
FORGE_SCAN_TRACE=1 python tools/trace_scan.py [op] [log2n]"""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["FORGE_SCAN_TRACE"] = "1"
import numpy as np, torch
from paper_2603_18695_b200 import capi, dev
op = int(sys.argv[1]) if len(sys.argv) > 1 else capi.F32_SUM
n = 1 << (int(sys.argv[2]) if len(sys.argv) > 2 else 28)
ws = dev.Workspace()
need = dev.workspace_bytes(capi.PRIM_SCAN, op, n)
tiles = n // 8192 + 2  # upper bound for any sub-tile count
ws.ensure(need + tiles * 64 + 4096)
src = dev.empty(op, n); dev.fill_synthetic(op, src, n, 3); dst = dev.empty(op, n, "S")
for _ in range(3):
    dev.scan(op, True, src, dst, n, ws)
torch.cuda.synchronize()
raw = ws.buf[need: need + (n // 8192) * 64].cpu().numpy().view(np.uint64).reshape(-1, 8).astype(np.int64)
t0 = raw[:, 0].min()
ph = raw[:, :5] - t0
d = {"tiles": len(raw), "span_us": float((ph[:, 4].max()) / 1e3)}
for i, name in enumerate(["claim->landed", "landed->pass1", "pass1->prefix", "prefix->end"]):
    x = (ph[:, i + 1] - ph[:, i]) / 1e3
    d[name] = {"mean_us": round(float(x.mean()), 3), "p50": round(float(np.median(x)), 3), "p90": round(float(np.percentile(x, 90)), 3), "max": round(float(x.max()), 3)}
life = (ph[:, 4] - ph[:, 0]) / 1e3
d["lifetime_us"] = {"mean": round(float(life.mean()), 3), "p50": round(float(np.median(life)), 3)}
# concurrency: tiles alive at the midpoint
mid = ph[:, 4].max() / 2
d["alive_at_mid"] = int(((ph[:, 0] <= mid) & (ph[:, 4] >= mid)).sum())
sms = raw[:, 5]
d["distinct_sms"] = int(len(np.unique(sms)))
# start rate
st = np.sort(ph[:, 0])
d["claims_per_us_mid"] = float(len(st) / (st[-1] - st[0]) * 1e3)
print(json.dumps(d, indent=1))
w = raw[:, 6]; p = raw[:, 7]
lb = (ph[:, 3] - ph[:, 2]) / 1e3
sel = w > 0  # look-back owners (every tile; the cluster kernel: leader sub-tiles)
print(json.dumps({"lookback_owners": int(sel.sum()), "windows_mean": float(w[sel].mean()),
                  "windows_p90": float(np.percentile(w[sel], 90)),
                  "poll_rounds_mean": float(p[sel].mean()),
                  "us_per_window": float((lb[sel] / np.maximum(w[sel], 1)).mean())}))
