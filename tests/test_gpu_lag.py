"""The lagged scan (include/forge/cuda/scan.cuh scan_lag_kernel, the default
for contiguous scans of >= 3 lags of full tiles (3 x 4 tiles per SM) with
sizeof(T) = sizeof(S) <= 8 and 16-byte carries: f32 affine with its f64
carry) at its boundaries, against the CPU oracle; the other ops in the same
tests (4- and 8-byte carries, 16-byte Mat2 elements) take the single-pass
kernel at the same sizes:

* the full-tile threshold (one below / at / above) and larger counts, plus
  sizes below it (the single-pass kernel);
* a partial last tile (the tail launch seeded with the full tiles' total);
* carry_in and total_out through the device-pointer layer (the sharded
  scan's carry), inclusive and exclusive;
* 16-byte elements (Mat2, single-pass since blockIdx tile order) next to
  quaternions (single-pass, 32-byte carry);
* one workspace reused across sizes whose layouts overlap (the tail's
  sub-workspace moves with the full-tile count).
"""
from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle as orc
from tests.helpers import TOL, assert_match

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
capi = pytest.importorskip("paper_2603_18695_b200.capi")
dev = pytest.importorskip("paper_2603_18695_b200.dev")
F = pytest.importorskip("paper_2603_18695_b200.forge")


def lag_tiles():
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    return sms * 4


def threshold():
    return 3 * lag_tiles()


def tile_elems(op):
    return 32768 // F.op_info(op)["t_size"]  # one 32 KB TMA tile


def to_np(t, dt):
    return t.cpu().numpy().view(np.uint8).view(dt)


def run(op, inclusive, x, ws, carry=None, want_total=False):
    n = len(x)
    src = torch.from_numpy(x.view(np.uint8).copy()).cuda()
    dst = dev.empty(op, n, "S")
    ss = F.s_dtype(op).itemsize
    cin = None
    if carry is not None:
        cin = torch.from_numpy(np.array([carry], dtype=F.s_dtype(op)).view(np.uint8).copy()).cuda()
    tot = torch.zeros(ss, dtype=torch.uint8, device="cuda") if want_total else None
    dev.scan(op, inclusive, src, dst, n, ws, carry_in=cin, total_out=tot)
    torch.cuda.synchronize()
    return to_np(dst, F.s_dtype(op)), (to_np(tot, F.s_dtype(op)) if want_total else None)


@pytest.mark.parametrize("op", [capi.AFFINE_F32, capi.MAT2_U32, capi.I32_SUM, capi.ARGMAX_F32I32])
@pytest.mark.parametrize("dt,extra", [(-1, 0), (0, 0), (1, 5), (500, 4097), (2000, 3), (-1000, 7)])
@pytest.mark.parametrize("inclusive", [True, False])
def test_lag_thresholds_and_tails(op, dt, extra, inclusive):
    tiles = threshold() + dt
    n = tiles * tile_elems(op) + extra
    x = orc.fill(op, n, 0x7A0 + tiles + extra)
    got, _ = run(op, inclusive, x, dev.Workspace())
    want, ex, sc = orc.scan(op, inclusive, x)
    assert_match(op, got, want, ex, sc, f"lagged scan tiles={tiles} extra={extra}")


@pytest.mark.parametrize("op", [capi.I32_SUM, capi.F32_SUM, capi.AFFINE_F32])
@pytest.mark.parametrize("inclusive", [True, False])
@pytest.mark.parametrize("extra", [0, 777])
def test_lag_carry_in_and_total_out(op, inclusive, extra):
    n = (threshold() + 50) * tile_elems(op) + extra
    x = orc.fill(op, n, 0x7B0 + op)
    c = orc.fill(op, 1, 0x7B1)[0]
    got, tot = run(op, inclusive, x, dev.Workspace(), carry=c, want_total=True)
    want, ex, sc = orc.scan(op, inclusive, x, carry=c)
    assert_match(op, got, want, ex, sc, "lagged scan with carry_in")
    # total_out = the inclusive total of carry + everything
    wi, exi, sci = orc.scan(op, True, x, carry=c)
    assert_match(op, tot, wi[-1:], exi[-1:], sci[-1:], "lagged scan total_out")


def test_lag_workspace_reuse_across_layouts():
    ws = dev.Workspace()
    op = capi.I32_SUM
    te = tile_elems(op)
    t0 = threshold()
    for tiles, extra in [(t0 + 300, 11), (200, 7), (t0 + 300, 11), (t0, 1), (t0 + 900, 3), (t0 + 1, 0),
                         (t0 + 300, 11)]:
        n = tiles * te + extra
        x = orc.fill(op, n, 0x7C0 + tiles)
        for inclusive in (True, False):
            got, _ = run(op, inclusive, x, ws)
            want, _, _ = orc.scan(op, inclusive, x)
            assert np.array_equal(got, want), (tiles, extra, inclusive)


def test_quaternion_single_pass_beside_lagged():
    # 32-byte f64 carry: the single-pass kernel (the lagged one spills)
    op = capi.QUAT_F32
    n = (threshold() + 10) * tile_elems(op) + 9
    x = orc.fill(op, n, 0x7D0)
    got, _ = run(op, True, x, dev.Workspace())
    want, ex, sc = orc.scan(op, True, x)
    assert_match(op, got, want, ex, sc, "quaternion scan")
    assert TOL[op] == 1e-5


def test_lag_ops_alternating_on_one_workspace():
    # lagged scans of different element / carry / ring-entry sizes alternate on
    # one workspace (the ring and the tile states move with the layout); each
    # output must equal its first (oracle-checked) launch bit for bit
    ws = dev.Workspace()
    ops = [capi.F32_SUM, capi.AFFINE_F32, capi.ARGMAX_F32I32, capi.MAT2_U32, capi.I32_SUM]
    cases = {}
    for op in ops:
        n = (threshold() + 300) * tile_elems(op) + 5
        x = orc.fill(op, n, 0x7F0 + op)
        got, _ = run(op, True, x, ws)
        want, ex, sc = orc.scan(op, True, x)
        assert_match(op, got, want, ex, sc, "alternating")
        cases[op] = (x, got)
    for _ in range(3):
        for op in ops:
            x, first = cases[op]
            got, _ = run(op, True, x, ws)
            if op in (capi.F32_SUM, capi.AFFINE_F32):
                want, ex, sc = orc.scan(op, True, x)
                assert_match(op, got, want, ex, sc, "alternating, again")
            else:
                assert got.tobytes() == first.tobytes(), op
