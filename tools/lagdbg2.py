"""Lagged-scan relaunch debug (development): alternating inputs on one
workspace, first mismatching index per launch."""
import sys
sys.path.insert(0, ".")
import numpy as np, torch
from oracle import oracle as orc
from paper_2603_18695_b200 import dev, capi
from paper_2603_18695_b200.forge import s_dtype
lib = capi.load()
op = int(sys.argv[1]) if len(sys.argv) > 1 else capi.I32_SUM
for n in [(1 << 22) + 17, 1 << 22]:
    ws = dev.Workspace()
    seeds = [0xAB1A, 0xAB1A ^ (0x5A5A << 40)]
    xs, want = [], []
    for k in range(2):
        x = dev.empty(op, n); dev.fill_synthetic(op, x, n, seeds[k]); xs.append(x)
        y = dev.empty(op, n, "S"); dev.scan(op, True, x, y, n, ws)
        got = y.cpu().numpy().view(np.uint8).view(s_dtype(op))
        print("check", k, orc.check_scan_synthetic(op, True, n, seeds[k], got, 1e-5)[0])
        want.append(y)
    for pert in [(0, 0), (0, 20000)]:
        lib.forge_set_schedule_perturbation(*pert)
        y = dev.empty(op, n, "S")
        for i in range(8):
            dev.scan(op, True, xs[i % 2], y, n, ws)
            d = (y.view(torch.int32) != want[i % 2].view(torch.int32)).nonzero()
            got = y.cpu().numpy().view(np.uint8).view(s_dtype(op))
            bad_orc = orc.check_scan_synthetic(op, True, n, seeds[i % 2], got, 1e-5)
            print(n, pert, i, "bad", d.numel(), d[:3].flatten().tolist() if d.numel() else "", "oracle", bad_orc, flush=True)
        lib.forge_set_schedule_perturbation(0, 0)
