"""Development: does the scan look-back ever read a predecessor's state before
the predecessor publishes it in the current launch?  (a) relax_scan_flag
mutant, alternating inputs; (b) product build with the epoch rewound so the
previous launch's states carry the current epoch."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2603_18695_b200 import capi, dev
lib = capi.load()
op = capi.I32_SUM
out = {}
for n in (1 << 20, 1 << 24, 1 << 26):
    xs = []
    for k in range(2):
        x = dev.empty(op, n); dev.fill_synthetic(op, x, n, 100 + k); xs.append(x)
    ws = dev.Workspace()
    want = []
    for k in range(2):
        y = dev.empty(op, n, "S"); dev.scan(op, True, xs[k], y, n, ws); want.append(y)
    y = dev.empty(op, n, "S")
    res = {}
    for relax in (0, 1):
        lib.forge_set_mutation_flags(relax, 0)
        bad = []
        for i in range(10):
            dev.scan(op, True, xs[i % 2], y, n, ws)
            bad.append(int((y.view(torch.int32) != want[i % 2].view(torch.int32)).sum().item()))
        lib.forge_set_mutation_flags(0, 0)
        res[f"relax{relax}"] = bad
    # rewind the epoch: ctrl word 2 of the workspace
    bad = []
    for i in range(10):
        e = ws.buf[8:12].clone()
        dev.scan(op, True, xs[i % 2], y, n, ws)
        torch.cuda.synchronize()
        ws.buf[8:12].copy_(e)  # next launch reuses this launch's epoch
        bad.append(int((y.view(torch.int32) != want[i % 2].view(torch.int32)).sum().item()))
    res["rewound"] = bad
    out[n] = res
print(json.dumps(out))
