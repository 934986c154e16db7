"""Single-pass scan tile order (development): FORGE_LIB=dev FORGE_SCAN_BLOCK_ORDER=0|1.
GB/s at 2^28 (median of 15) and 2^23, plus oracle checks, for the ops of the
single-pass tile kernel (carries <= 8 bytes) and of the lagged kernel (affine, Mat2)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import oracle as orc  # noqa: E402
from paper_2603_18695_b200 import capi, dev  # noqa: E402
from paper_2603_18695_b200.forge import op_info, s_dtype  # noqa: E402


def t(fn, reps=15):
    s = torch.cuda.current_stream()
    fn()
    torch.cuda.synchronize()
    ev = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        fn()
        b.record(s)
        ev.append((a, b))
    torch.cuda.synchronize()
    x = sorted(a.elapsed_time(b) for a, b in ev)
    return x[len(x) // 2]


ws = dev.Workspace()
out = {"block_order": os.environ.get("FORGE_SCAN_BLOCK_ORDER", "default")}
for name in ("F32_SUM", "I32_SUM", "ARGMAX_F32I32", "I64_SUM", "AFFINE_F32", "MAT2_U32"):
    op = getattr(capi, name)
    inf = op_info(op)
    for lg in (28, 23):
        lg -= 1 if inf["t_size"] >= 16 else 0
        n = 1 << lg
        src = dev.empty(op, n)
        dev.fill_synthetic(op, src, n, 3)
        dst = dev.empty(op, n, "S")
        for incl in (True, False):
            ms = t(lambda: dev.scan(op, incl, src, dst, n, ws))
            out[f"{name}_2^{lg}_{'incl' if incl else 'excl'}"] = round(n * (inf["t_size"] + inf["s_size"]) / ms / 1e6, 1)
        del src, dst
    # correctness: ragged size, relaunches on one workspace
    n = (1 << 24) + 4097
    src = dev.empty(op, n)
    dev.fill_synthetic(op, src, n, 77)
    dst = dev.empty(op, n, "S")
    bad = 0
    for incl in (True, False):
        for _ in range(3):
            dev.scan(op, incl, src, dst, n, ws)
            got = dst.cpu().numpy().view(np.uint8).view(s_dtype(op))
            bad += orc.check_scan_synthetic(op, incl, n, 77, got, 1e-5)[0]
    out[f"{name}_bad"] = bad
    del src, dst
print(json.dumps(out))
