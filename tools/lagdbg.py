import sys; sys.path.insert(0, ".")
import numpy as np, torch
from oracle import oracle as orc
from paper_2603_18695_b200 import dev, capi
from paper_2603_18695_b200.forge import s_dtype
for op in [10, 0, 12]:
  for incl in [True, False]:
    for n in [1000003, 1 << 20, 3 * 1024 * 1024 + 5]:
        x = orc.fill(op, n, 0x6B0 + op)
        t = torch.from_numpy(x.view(np.uint8).copy()).cuda()
        y = dev.empty(op, n, "S")
        dev.scan(op, incl, t, y, n, dev.Workspace())
        torch.cuda.synchronize()
        got = y.cpu().numpy().view(s_dtype(op))
        want, ex, sc = orc.scan(op, incl, x)
        if orc.ncomp(op):
            ok, rel = orc.within(op, got, ex, sc, 1e-5)
        else:
            ok, rel = np.array_equal(got.view(np.uint8), want.view(np.uint8)), 0
        print(op, incl, n, ok, rel, flush=True)
