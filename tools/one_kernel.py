"""Runs one primitive a few times (for ncu captures). usage: one_kernel.py mapreduce|scan|gevm|gemv|copy [op]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2603_18695_b200 import capi, dev
what = sys.argv[1]
ws = dev.Workspace()
if what == "mapreduce":
    op = int(sys.argv[2]) if len(sys.argv) > 2 else capi.F32_SUMSQ
    n = 1 << 30
    x = dev.empty(op, n); dev.fill_synthetic(op, x, n, 1)
    out = torch.zeros(16, dtype=torch.uint8, device="cuda")
    for _ in range(3): dev.mapreduce(op, x, n, out, ws)
elif what == "scan":
    op = int(sys.argv[2]) if len(sys.argv) > 2 else capi.F32_SUM
    n = 1 << 28
    x = dev.empty(op, n); dev.fill_synthetic(op, x, n, 1); y = dev.empty(op, n, "S")
    for _ in range(3): dev.scan(op, True, x, y, n, ws)
elif what == "copy":
    nb = 2 << 30
    a = torch.empty(nb, dtype=torch.uint8, device="cuda"); b = torch.empty(nb, dtype=torch.uint8, device="cuda")
    for _ in range(3): dev.copy(a, b, nb)
else:
    op = int(sys.argv[2]) if len(sys.argv) > 2 else capi.MV_F32_PLUS_TIMES
    nn = 16384
    A = dev.empty(op, nn * nn); dev.fill_synthetic(op, A, nn * nn, 5)
    x = dev.empty(op, nn); dev.fill_synthetic(op, x, nn, 6); y = dev.empty(op, nn, "S")
    fn = dev.matvec if what == "gevm" else dev.vecmat
    for _ in range(3): fn(op, A, nn, nn, x, y, ws)
torch.cuda.synchronize()
