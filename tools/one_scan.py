import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2603_18695_b200 import capi, dev
op = int(sys.argv[1]) if len(sys.argv) > 1 else capi.F32_SUM
n = 1 << 28
ws = dev.Workspace()
src = dev.empty(op, n); dev.fill_synthetic(op, src, n, 3); dst = dev.empty(op, n, "S")
for _ in range(3):
    dev.scan(op, True, src, dst, n, ws)
torch.cuda.synchronize()
