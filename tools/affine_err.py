"""Worst |got - exact| / scale of the affine scan at several sizes (development
tool): the B200 kernel on the GPU vs the streaming oracle, plus the reference
VM's own error where the VM is built (CPU only)."""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
from oracle import oracle as orc  # noqa: E402

op = 10
rows = []
if "--ref" in sys.argv:
    for n in [4097, 100_003, 1 << 20]:
        seed = 0x5EED0020 + op
        x = orc.fill(op, n, seed)
        got, _ = orc.ref_scan(op, True, x, backend=orc.THREADS)
        _, ex, sc = orc.scan(op, True, x)
        rows.append({"who": "reference_vm", "n": n, "worst": orc.within(op, got, ex, sc, 1e-5)[1]})
else:
    import torch  # noqa: F401
    from paper_2603_18695_b200 import dev
    from paper_2603_18695_b200.forge import s_dtype
    for n in [4097, 100_003, 1 << 20, 1 << 24, 1 << 28]:
        for incl in (True, False):
            seed = 0x5EED0020 + op
            x = dev.empty(op, n)
            dev.fill_synthetic(op, x, n, seed)
            y = dev.empty(op, n, "S")
            dev.scan(op, incl, x, y, n, dev.Workspace())
            got = y.cpu().numpy().view(np.uint8).view(s_dtype(op))
            bad, worst = orc.check_scan_synthetic(op, incl, n, seed, got, 1e-5)
            rows.append({"who": "b200", "n": n, "inclusive": incl, "bad_at_1e-5": bad, "worst": worst})
for r in rows:
    print(json.dumps(r))
