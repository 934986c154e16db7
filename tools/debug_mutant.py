"""Development: relaxed-protocol mutant vs schedule perturbation, per op:
number of mismatching elements per launch (alternating inputs, one workspace)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2603_18695_b200 import capi, dev
lib = capi.load()
out = {}
for op in (capi.I32_SUM, capi.F32_SUM, capi.MAT2_U32):
    n = (1 << 22) + 17
    xs = []
    for k in range(2):
        x = dev.empty(op, n); dev.fill_synthetic(op, x, n, 0xAB1A ^ (k * 0x5A5A << 40)); xs.append(x)
    ws = dev.Workspace()
    want = []
    for k in range(2):
        y = dev.empty(op, n, "S"); dev.scan(op, True, xs[k], y, n, ws); want.append(y)
    y = dev.empty(op, n, "S")
    res = {}
    for relax, seed, ns in ((0, 0, 0), (1, 0, 0), (0, 0x5EED, 20000), (1, 0x5EED, 20000), (1, 0x5EED, 100000)):
        lib.forge_set_mutation_flags(relax, 0)
        lib.forge_set_schedule_perturbation(seed, ns)
        bad = []
        for i in range(6):
            y.fill_(0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            dev.scan(op, True, xs[i % 2], y, n, ws)
            e1.record(); torch.cuda.synchronize()
            bad.append((int((y != want[i % 2]).sum().item()), round(e0.elapsed_time(e1), 3)))
        lib.forge_set_mutation_flags(0, 0); lib.forge_set_schedule_perturbation(0, 0)
        res[f"relax{relax}_seed{seed}_{ns}"] = bad
    out[op] = res
print(json.dumps(out, indent=1))
