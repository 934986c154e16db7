"""Per-tile event timing of the carry-chain scan kernel (development tool).
python tools/trace_chain.py [op] [log2n]   (sets FORGE_SCAN_PATH=chain, FORGE_SCAN_TRACE=1;
needs a `make EXPERIMENTS=1` build)"""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["FORGE_SCAN_TRACE"] = "1"
os.environ.setdefault("FORGE_SCAN_PATH", "chain")
import numpy as np, torch
from paper_2603_18695_b200 import capi, dev
op = int(sys.argv[1]) if len(sys.argv) > 1 else capi.F32_SUM
n = 1 << (int(sys.argv[2]) if len(sys.argv) > 2 else 28)
ws = dev.Workspace()
need = dev.workspace_bytes(capi.PRIM_SCAN, op, n)
tiles = n // 8192
ws.ensure(need + (tiles + 2) * 64 + 2048 * 32 + 4096)
src = dev.empty(op, n); dev.fill_synthetic(op, src, n, 3); dst = dev.empty(op, n, "S")
for _ in range(3):
    dev.scan(op, True, src, dst, n, ws)
torch.cuda.synchronize()
raw = ws.buf[need: need + tiles * 64].cpu().numpy().view(np.uint64).reshape(-1, 8).astype(np.int64)
t0 = raw[:, 0].min()
ev = (raw[:, :6] - t0) / 1e3
names = ["issue", "partial", "chain", "fetched", "scan_start", "scan_end"]
d = {"tiles": len(raw), "span_us": float(ev[:, 5].max())}
for i in range(5):
    x = ev[:, i + 1] - ev[:, i]
    d[names[i] + "->" + names[i + 1]] = {"mean": round(float(x.mean()), 3), "p50": round(float(np.median(x)), 3),
                                          "p90": round(float(np.percentile(x, 90)), 3)}
# chain throughput over the middle half
ch = np.sort(ev[:, 2]); q = len(ch) // 4
d["chain_tiles_per_us_mid"] = float((2 * q) / (ch[3 * q] - ch[q]))
pa = np.sort(ev[:, 1])
d["partial_tiles_per_us_mid"] = float((2 * q) / (pa[3 * q] - pa[q]))
# chain lag behind the partial frontier (tiles) at mid time
mid = ev[:, 5].max() / 2
d["partials_done_at_mid"] = int((ev[:, 1] <= mid).sum())
d["chain_done_at_mid"] = int((ev[:, 2] <= mid).sum())
d["scans_done_at_mid"] = int((ev[:, 5] <= mid).sum())
r = raw[:, 7]
rounds = r >> 8; nr = r & 255
d["chain_rounds_total"] = int(rounds.max())
d["rows_per_round_mean"] = float(np.mean([nr[rounds == k][0] for k in np.unique(rounds)[:2000]]))
d["us_per_round"] = float((ev[:, 2].max() - ev[:, 2].min()) / max(1, rounds.max()))
rr = ws.buf[need + tiles * 64: need + tiles * 64 + 2048 * 32].cpu().numpy().view(np.uint64).reshape(-1, 4).astype(np.int64)
rr = rr[1:int(rounds.max()) + 1]
d["round_poll_us"] = float(np.median(rr[:, 1] - rr[:, 0]) / 1e3)
d["round_proc_us"] = float(np.median(rr[:, 2] - rr[:, 1]) / 1e3)
d["round_nready_median"] = float(np.median(rr[:, 3]))
print(json.dumps(d, indent=1))
