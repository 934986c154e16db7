"""Small run of every sm_100a kernel family for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck).  usage: python tools/sanitize_run.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2603_18695_b200 import capi, dev  # noqa: E402

ws = dev.Workspace()
out = torch.zeros(16, dtype=torch.uint8, device="cuda")
for op in (capi.F32_SUM, capi.I32_MAX, capi.AFFINE_F32, capi.MAT2_U32, capi.UF8_F32_SUM):
    for n in (1, 1000, 3 * 8192 + 17, 70_000):
        x = dev.empty(op, n)
        dev.fill_synthetic(op, x, n, 11)
        y = dev.empty(op, n, "S")
        for incl in (True, False):
            try:
                dev.scan(op, incl, x, y, n, ws)
            except Exception as e:  # UF8 scans are not on the menu
                if "Unsupported" not in str(e):
                    raise
        try:
            dev.mapreduce(op, x, n, out, ws)
        except Exception as e:  # non-commutative ops: ordered reduce instead
            if "commutative" not in str(e):
                raise
        dev.reduce_ordered(op, x, n, out, ws)
# the lagged scan: with the DEV library and FORGE_SCAN_LAG=16 it takes scans of
# >= 128 full tiles (140 tiles + a tail here; argmax past the 2048-slot ring)
if os.environ.get("FORGE_LIB") == "dev" and os.environ.get("FORGE_SCAN_LAG"):
    from paper_2603_18695_b200.forge import op_info
    for op, tiles in ((capi.F32_SUM, 140), (capi.ARGMAX_F32I32, 140), (capi.AFFINE_F32, 140),
                      (capi.MAT2_U32, 140), (capi.ARGMAX_F32I32, 2100)):
        n = tiles * (32768 // op_info(op)["t_size"]) + 17
        x = dev.empty(op, n)
        dev.fill_synthetic(op, x, n, 12)
        y = dev.empty(op, n, "S")
        for incl in (True, False):
            dev.scan(op, incl, x, y, n, ws)
        del x, y
for op in (capi.MV_F32_PLUS_TIMES, capi.MV_F32_MIN_PLUS):
    for n, p in ((257, 129), (4096, 7), (64, 2048)):
        A = dev.empty(op, n * p)
        dev.fill_synthetic(op, A, n * p, 3)
        xv = dev.empty(op, max(n, p))
        dev.fill_synthetic(op, xv, max(n, p), 4)
        yv = dev.empty(op, max(n, p), "S")
        dev.matvec(op, A, n, p, xv, yv, ws)
        dev.vecmat(op, A, n, p, xv, yv, ws)
from paper_2603_18695_b200 import forge as F  # noqa: E402
r = F.run_litmus("blocks=2 cells=2\nB0: st 0 =1\nB0: st 1 rel =1\nB1: ld 1 acq\nB1: ld 0\n", 0, 256)
assert r["faults"] == 0
a = torch.empty(1 << 20, dtype=torch.uint8, device="cuda")
b = torch.empty(1 << 20, dtype=torch.uint8, device="cuda")
a.fill_(7)
dev.copy(a, b, 1 << 20)
torch.cuda.synchronize()
print("sanitize_run ok")
