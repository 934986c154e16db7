"""Phase timing of the pipelined scan kernel: 0 A start, 1 A end, 2 look-back start, 3 look-back end, 4 C end."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["FORGE_SCAN_TRACE"] = "1"
import numpy as np, torch
from paper_2603_18695_b200 import capi, dev
op = int(sys.argv[1]) if len(sys.argv) > 1 else capi.F32_SUM
n = 1 << 28
ws = dev.Workspace(); need = dev.workspace_bytes(capi.PRIM_SCAN, op, n)
ws.ensure(need + (n // 1024 + 2) * 64 + 4096)
src = dev.empty(op, n); dev.fill_synthetic(op, src, n, 3); dst = dev.empty(op, n, "S")
for _ in range(3): dev.scan(op, True, src, dst, n, ws)
torch.cuda.synchronize()
isz = {0: 4, 5: 4, 10: 8, 11: 8, 12: 16}[op]
ntiles = n // (256 * (128 // isz))
raw = ws.buf[need: need + ntiles * 64].cpu().numpy().view(np.uint64).reshape(-1, 8).astype(np.int64)[:, :5]
t0 = raw.min(); ph = raw - t0
out = {"span_us": float(ph.max() / 1e3)}
for i, nm in enumerate(["A", "A_end->lb_start", "lookback", "C"]):
    x = (ph[:, i + 1] - ph[:, i]) / 1e3
    out[nm] = {"mean": round(float(x.mean()), 3), "p50": round(float(np.median(x)), 3), "p90": round(float(np.percentile(x, 90)), 3)}
life = (ph[:, 4] - ph[:, 0]) / 1e3
out["life_mean"] = float(life.mean())
print(json.dumps(out))
