"""Round-2 parity holes (VERDICT r01 "What's weak" #1):

* special values: f32 max / min and arg-max over data with NaN (random payloads
  and signs), +-inf and signed zeros are bit-exact against the oracle for every
  tree shape — the operators are order-independent by definition
  (include/forge/algebra.hpp fmax_total / fmin_total / argmax_combine);
* empty inputs (n = 0) through both C-ABI layers;
* one workspace shared by every primitive and several matrix shapes in turn
  (the library re-zeroes a workspace whose layout changes: cuda::ws_claim);
* dev.Workspace growth on a non-current stream.
"""
from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle as orc
from tests.helpers import SIZES, assert_match, seed_for

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
capi = pytest.importorskip("paper_2603_18695_b200.capi")
dev = pytest.importorskip("paper_2603_18695_b200.dev")
F = pytest.importorskip("paper_2603_18695_b200.forge")

SPECIAL_OPS = [capi.F32_MAX, capi.F32_MIN, capi.ARGMAX_F32I32]


def to_np(t, dtype):
    return t.cpu().numpy().view(np.uint8).view(dtype)


@pytest.fixture(scope="module")
def m():
    mach = F.Machine(0)
    yield mach
    mach.close()


def test_special_value_generator_has_specials():
    x = orc.fill(capi.F32_MAX, 1 << 20, 77, variant=2)
    bits = x.view(np.uint32)
    assert np.isnan(x).sum() >= 4 and np.isinf(x).sum() >= 4
    assert (bits == 0x80000000).sum() > 1000 and (bits == 0).sum() > 1000
    assert len(set(bits[np.isnan(x)].tolist())) > 1  # several NaN payloads


@pytest.mark.parametrize("op", SPECIAL_OPS)
def test_device_generator_special_values(op):
    n = 100_003
    t = dev.empty(op, n)
    dev.fill_synthetic(op, t, n, 4321, index_base=7, variant=2)
    assert np.array_equal(to_np(t, orc.t_dtype(op)).view(np.uint8),
                          orc.fill(op, n, 4321, variant=2, index_base=7).view(np.uint8))


@pytest.mark.parametrize("op", SPECIAL_OPS)
@pytest.mark.parametrize("n", [1, 2, 33, 4097, 100_000, 1 << 20, 3_000_001])
def test_mapreduce_special_values_bit_exact(m, op, n):
    x = orc.fill(op, n, seed_for(op, n, 2), variant=2)
    b = F.create_buffer(m, op, n)
    m.write(b, x)
    ws = F.make_mapreduce_workspace(m, op)
    got, rep = F.mapreduce(m, F.make_semiring(op), F.make_view(m, b), ws)
    want, ex, sc = orc.mapreduce(op, x)
    assert rep.ok
    assert_match(op, np.array([got], dtype=F.s_dtype(op)), np.array([want]), ex, sc, f"special n={n}")
    F.release(m, ws)
    m.destroy_buffer(b)


@pytest.mark.parametrize("op", SPECIAL_OPS)
@pytest.mark.parametrize("n", [1, 257, 8193, 100_000, 1 << 20])
@pytest.mark.parametrize("inclusive", [True, False])
def test_scan_special_values_bit_exact(m, op, n, inclusive):
    # NaN is about 1 in 2^15 elements: the prefixes before the first NaN carry
    # +-0 / +-inf ties; every later prefix is the canonical NaN (or, for the
    # arg-max, the first NaN element with its own payload).
    x = orc.fill(op, n, seed_for(op, n, inclusive, 2), variant=2)
    a = F.create_buffer(m, op, n)
    d = F.create_buffer(m, op, n, which="S")
    m.write(a, x)
    ws = F.make_scan_workspace(m, op, n)
    rep = F.scan(m, F.make_semiring(op), F.make_view(m, a), F.make_view(m, d), inclusive, ws)
    assert rep.ok
    want, ex, sc = orc.scan(op, inclusive, x)
    assert_match(op, m.read(d, n, F.s_dtype(op)), want, ex, sc, f"special scan n={n}")
    F.release(m, ws)
    m.destroy_buffer(a)
    m.destroy_buffer(d)


@pytest.mark.parametrize("op", [capi.MV_F32_MIN_PLUS, capi.MV_F32_MAX_PLUS])
@pytest.mark.parametrize("which", ["matvec", "vecmat"])
def test_tropical_matrix_signed_zero_ties(op, which):
    # min-plus / max-plus with many +-0 and small-integer ties (no NaN / inf:
    # f = a + b of two infinities would make a host- and device-specific NaN
    # before any op canonicalises it)
    rng = np.random.default_rng(op)
    n, p = 3000, 517
    A = rng.integers(-2, 3, n * p).astype(np.float32) * np.float32(0.5)
    A[rng.random(n * p) < 0.3] = np.float32(-0.0)
    x = rng.integers(-2, 3, n if which == "matvec" else p).astype(np.float32)
    x[rng.random(len(x)) < 0.3] = np.float32(-0.0)
    Ad, xd = torch.from_numpy(A.view(np.uint8).copy()).cuda(), torch.from_numpy(x.view(np.uint8).copy()).cuda()
    outn = p if which == "matvec" else n
    y = torch.zeros(outn * 4, dtype=torch.uint8, device="cuda")
    ws = dev.Workspace()
    (dev.matvec if which == "matvec" else dev.vecmat)(op, Ad, n, p, xd, y, ws)
    want, _, _ = (orc.matvec if which == "matvec" else orc.vecmat)(op, A, n, p, x)
    assert np.array_equal(to_np(y, np.float32).view(np.uint32), want.view(np.uint32))


# ---------------------------------------------------------------------------
# empty inputs (SPEC.md:512 includes n = 0)

@pytest.mark.parametrize("op", [capi.F32_SUM, capi.I32_MAX, capi.MAT2_U32, capi.AFFINE_F32, capi.UF8_F32_SUM])
def test_empty_inputs_both_layers(m, op):
    a = F.create_buffer(m, op, 4)
    d = F.create_buffer(m, op, 4, which="S")
    sentinel = np.full(4 * F.op_info(op)["s_size"], 0xAB, np.uint8)
    m.write(d, sentinel.view(F.s_dtype(op)))
    ws = F.make_scan_workspace(m, op, 0)
    for inclusive in (True, False):
        rep = F.scan(m, F.make_semiring(op), F.View(a, 0, 0, 1), F.View(d, 0, 0, 1), inclusive, ws)
        assert rep.ok
    assert np.array_equal(m.read(d, 4, F.s_dtype(op)).view(np.uint8), sentinel)  # nothing written
    # device-pointer layer: n = 0 scan is a no-op; n = 0 mapreduce writes the identity
    src = dev.empty(op, 4)
    dst = torch.full((4 * F.op_info(op)["s_size"],), 0xAB, dtype=torch.uint8, device="cuda")
    w = dev.Workspace()
    dev.scan(op, True, src, dst, 0, w)
    torch.cuda.synchronize()
    assert bool((dst == 0xAB).all())
    if F.op_info(op)["commutative"]:
        out = torch.zeros(16, dtype=torch.uint8, device="cuda")
        dev.mapreduce(op, src, 0, out, w)
        want, _, _ = orc.mapreduce(op, np.zeros(0, orc.t_dtype(op)))
        got = out[: F.op_info(op)["s_size"]].cpu().numpy().view(F.s_dtype(op))
        assert got.view(np.uint8).tobytes() == np.atleast_1d(want).view(np.uint8).tobytes()


# ---------------------------------------------------------------------------
# one workspace for everything

def test_one_dev_workspace_for_every_primitive_and_shape():
    ws = dev.Workspace()
    rng = np.random.default_rng(5)
    cases = []
    # exact ops so every check is bitwise
    for n in (300_007, 5_000_000):
        op = capi.I32_SUM
        x = orc.fill(op, n, 11 + n)
        cases.append(("scan", op, n, x))
        cases.append(("mapreduce", capi.I32_MAX, n, orc.fill(capi.I32_MAX, n, 12 + n)))
        cases.append(("reduce_ordered", capi.MAT2_U32, n // 8, orc.fill(capi.MAT2_U32, n // 8, 13 + n)))
    shapes = [(200_003, 8), (1000, 60_000), (4096, 4096), (64, 3), (100_000, 40)]
    for n, p in shapes:
        op = capi.MV_I32_PLUS_TIMES
        A = orc.fill(op, n * p, n + p)
        cases.append(("matvec", op, (n, p), (A, orc.fill(op, n, 7))))
        cases.append(("vecmat", op, (n, p), (A, orc.fill(op, p, 8))))
    order = list(range(len(cases))) * 2
    rng.shuffle(order)
    for k in order:
        kind, op, n, data = cases[k]
        if kind == "scan":
            x = torch.from_numpy(data.view(np.uint8).copy()).cuda()
            y = dev.empty(op, n, "S")
            dev.scan(op, True, x, y, n, ws)
            want, _, _ = orc.scan(op, True, data)
            assert np.array_equal(to_np(y, np.int32), want), kind
        elif kind in ("mapreduce", "reduce_ordered"):
            x = torch.from_numpy(data.view(np.uint8).copy()).cuda()
            out = torch.zeros(16, dtype=torch.uint8, device="cuda")
            (dev.mapreduce if kind == "mapreduce" else dev.reduce_ordered)(op, x, n, out, ws)
            want, _, _ = orc.mapreduce(op, data) if kind == "mapreduce" else orc.scan(op, True, data)
            want = np.atleast_1d(want)[-1:] if kind == "reduce_ordered" else np.atleast_1d(want)
            ss = F.op_info(op)["s_size"]
            assert out[:ss].cpu().numpy().tobytes() == want.view(np.uint8).tobytes(), kind
        else:
            (nn, pp), (A, x) = n, data
            Ad = torch.from_numpy(A.view(np.uint8).copy()).cuda()
            xd = torch.from_numpy(x.view(np.uint8).copy()).cuda()
            outn = pp if kind == "matvec" else nn
            y = torch.zeros(outn * 4, dtype=torch.uint8, device="cuda")
            (dev.matvec if kind == "matvec" else dev.vecmat)(op, Ad, nn, pp, xd, y, ws)
            want, _, _ = (orc.matvec if kind == "matvec" else orc.vecmat)(op, A, nn, pp, x)
            assert np.array_equal(to_np(y, np.int32), want), (kind, nn, pp)


def test_dev_workspace_grows_on_a_side_stream():
    side = torch.cuda.Stream()
    ws = dev.Workspace()
    op = capi.I32_SUM
    for n in (1000, 1 << 20, 1 << 24):  # every call grows the workspace
        x = dev.empty(op, n)
        dev.fill_synthetic(op, x, n, 3 + n)
        y = dev.empty(op, n, "S")
        with torch.cuda.stream(side):
            dev.scan(op, True, x, y, n, ws, stream=side)
        side.synchronize()
        bad, _ = orc.check_scan_synthetic(op, True, n, 3 + n, to_np(y, np.int32), 0)
        assert bad == 0
