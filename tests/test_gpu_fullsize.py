"""BASELINE-size parity through the device-pointer
C-ABI, with inputs made on the GPU by the synthetic generator and checked by
the STREAMING oracle (oracle/oracle.c regenerates every input element from the
same splitmix64 counter, so no input is materialised on the host)."""
from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle as orc
from tests.helpers import TOL

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
capi = pytest.importorskip("paper_2603_18695_b200.capi")
dev = pytest.importorskip("paper_2603_18695_b200.dev")
F = pytest.importorskip("paper_2603_18695_b200.forge")


def to_np(t: "torch.Tensor", dtype) -> np.ndarray:
    return t.cpu().numpy().view(np.uint8).view(dtype)


@pytest.mark.parametrize("op", [capi.F32_SUMSQ, capi.I32_MAX, capi.F32_SUM, capi.UF8_F32_SUM])
def test_mapreduce_2pow30(op):
    n = 1 << 30
    seed = 0x5EED0010 + op
    x = dev.empty(op, n)
    dev.fill_synthetic(op, x, n, seed)
    out = torch.zeros(16, dtype=torch.uint8, device="cuda")
    ws = dev.Workspace()
    dev.mapreduce(op, x, n, out, ws)
    got = to_np(out[: F.s_dtype(op).itemsize], F.s_dtype(op))
    want, ex, sc = orc.mapreduce_synthetic(op, n, seed)
    if orc.ncomp(op):
        ok, rel = orc.within(op, got, ex, sc, TOL[op])
        assert ok, rel
    else:
        assert got[0] == want


@pytest.mark.parametrize("op,variant", [(capi.AFFINE_F32, 0), (capi.ARGMAX_F32I32, 0), (capi.ARGMAX_F32I32, 1),
                                        (capi.F32_SUM, 0)])
@pytest.mark.parametrize("inclusive", [True, False])
def test_scan_2pow28(op, variant, inclusive):
    n = 1 << 28
    seed = 0x5EED0020 + op
    x = dev.empty(op, n)
    dev.fill_synthetic(op, x, n, seed, variant=variant)
    y = dev.empty(op, n, "S")
    ws = dev.Workspace()
    dev.scan(op, inclusive, x, y, n, ws)
    got = to_np(y, F.s_dtype(op))
    del x, y
    bad, worst = orc.check_scan_synthetic(op, inclusive, n, seed, got, TOL.get(op, 1e-5), variant=variant)
    assert bad == 0, f"{bad} mismatching elements, worst err/scale {worst:.3e}"


def test_scan_sharded_emulation_carry_in():
    # C5 on one GPU: G contiguous shards, shard totals by the order-preserving
    # reduce, rank-order exclusive fold -> carry-in, seeded local scans; must
    # equal the single-pass scan bit for bit (exact op) — the same code path the
    # multi-GPU exchange uses (paper_2603_18695_b200/sharded.py).
    op, n, G = capi.MAT2_U32, 3_000_017, 4
    x = dev.empty(op, n)
    dev.fill_synthetic(op, x, n, 77)
    sz = F.t_dtype(op).itemsize
    ref = dev.empty(op, n, "S")
    ws = dev.Workspace()
    dev.scan(op, False, x, ref, n, ws)
    bounds = [n * g // G for g in range(G + 1)]
    totals = torch.zeros(G * sz, dtype=torch.uint8, device="cuda")
    for g in range(G):
        lo, hi = bounds[g], bounds[g + 1]
        dev.reduce_ordered(op, x.data_ptr() + lo * sz, hi - lo, totals.data_ptr() + g * sz, ws)
    out = dev.empty(op, n, "S")
    carry = torch.zeros(sz, dtype=torch.uint8, device="cuda")
    has = torch.zeros(1, dtype=torch.int32, device="cuda")
    for g in range(G):
        lo, hi = bounds[g], bounds[g + 1]
        dev.fold(op, totals, G, carry, exclusive_upto=g, has_out=has)
        torch.cuda.synchronize()
        cin = carry if int(has.item()) else None
        dev.scan(op, False, x.data_ptr() + lo * sz, out.data_ptr() + lo * sz, hi - lo, ws, carry_in=cin)
    torch.cuda.synchronize()
    # against the streaming oracle (exact op: bit for bit), then the single-pass scan
    bad, _ = orc.check_scan_synthetic(op, False, n, 77, to_np(out, F.s_dtype(op)), 0.0)
    assert bad == 0, f"{bad} elements of the G-shard scan differ from the oracle"
    assert torch.equal(out, ref)


@pytest.mark.parametrize("op", [capi.F32_SUM, capi.MAT2_U32])
def test_native_group_c5_emulated(op):
    # BASELINE C5's sharded exclusive scan + mapreduce through the native group
    # layer (forge_sharded_*), G = 4 emulated shards on one GPU, shards generated
    # in place (index_base = shard start), checked by the streaming oracle.
    from paper_2603_18695_b200 import group
    n = (1 << 28) if op == capi.F32_SUM else (1 << 26)
    seed, G = 0x5EED0C05, 4
    sz, ss = F.t_dtype(op).itemsize, F.s_dtype(op).itemsize
    with group.Group([0] * G) as g:
        src, dst, ns = [], [], []
        for r in range(G):
            lo, hi = group.shard_range(n, r, G)
            t = torch.empty((hi - lo) * sz, dtype=torch.uint8, device="cuda")
            dev.fill_synthetic(op, t, hi - lo, seed, index_base=lo)
            src.append(t)
            dst.append(torch.empty((hi - lo) * ss, dtype=torch.uint8, device="cuda"))
            ns.append(hi - lo)
        g.scan(op, False, src, dst, ns)
        got = np.concatenate([d.cpu().numpy() for d in dst]).view(F.s_dtype(op))
        bad, worst = orc.check_scan_synthetic(op, False, n, seed, got, TOL.get(op, 0.0))
        assert bad == 0, f"{bad} mismatches, worst {worst:.3e}"
        if op == capi.F32_SUM:
            total = np.frombuffer(g.mapreduce(op, src, ns), dtype=np.float32)
            want, ex, sc = orc.mapreduce_synthetic(op, n, seed)
            ok, rel = orc.within(op, total, ex, sc, TOL[op])
            assert ok, rel


@pytest.mark.parametrize("which", ["matvec", "vecmat"])
@pytest.mark.parametrize("op", [capi.MV_F32_PLUS_TIMES, capi.MV_F32_MIN_PLUS])
def test_matrix_16384(which, op):
    nn = 16384
    A = dev.empty(op, nn * nn)
    dev.fill_synthetic(op, A, nn * nn, 5)
    x = dev.empty(op, nn)
    dev.fill_synthetic(op, x, nn, 6)
    y = dev.empty(op, nn, "S")
    ws = dev.Workspace()
    (dev.matvec if which == "matvec" else dev.vecmat)(op, A, nn, nn, x, y, ws)
    got = to_np(y, np.float32)
    An, xn = to_np(A, np.float32), to_np(x, np.float32)
    want, ex, sc = (orc.matvec if which == "matvec" else orc.vecmat)(op, An, nn, nn, xn)
    if orc.ncomp(op):
        ok, rel = orc.within(op, got, ex, sc, TOL[op])
        assert ok, rel
    else:
        assert np.array_equal(got, want)


def test_device_generator_matches_host_generator():
    for op in [0, 4, 5, 9, 10, 11, 12, 13, 14, 32, 37]:
        for variant in (0, 1):
            n = 10_007
            t = dev.empty(op, n)
            dev.fill_synthetic(op, t, n, 1234, index_base=99, variant=variant)
            got = to_np(t, orc.t_dtype(op))
            want = orc.fill(op, n, 1234, variant=variant, index_base=99)
            assert np.array_equal(got.view(np.uint8), want.view(np.uint8)), (op, variant)


def test_uf8_decode_exhaustive_bitwise():
    # The device decode (reciprocal + FMA correction) equals the correctly
    # rounded -1 + 2c/255 for all 256 codes: inclusive scan of a single element
    # outputs f(x0) with no further rounding.
    m = F.Machine(0)
    a = F.create_buffer(m, capi.UF8_F32_SUM, 1)
    d = F.create_buffer(m, capi.UF8_F32_SUM, 1, which="S")
    ws = F.make_scan_workspace(m, capi.UF8_F32_SUM, 1)
    L = orc.lib()
    for c in range(256):
        m.write(a, np.array([c], np.uint8))
        F.scan(m, F.make_semiring(capi.UF8_F32_SUM), F.make_view(m, a), F.make_view(m, d), True, ws)
        got = m.read(d, 1, np.float32)[0]
        assert np.float32(got) == np.float32(L.orc_uf8_decode(c)), c
    m.close()


def test_c5_sharded_scan_and_mapreduce_2pow33():
    # BASELINE C5 at G = 1 box-local shards: n = 2^33 f32 (32 GiB in, 32 GiB out),
    # exclusive scan and mapreduce through the multi-GPU exchange code path
    # (order-preserving shard totals -> rank-order fold -> carry-seeded scans),
    # G = 4 shards emulated on one GPU.  Outputs are checked by the streaming
    # oracle at 4096 random positions plus every shard boundary +-1 (the
    # outputs never leave the device in full).
    op, n, G = capi.F32_SUM, 1 << 33, 4
    seed = 0x5EED0C05
    sz = 4
    x = dev.empty(op, n)
    dev.fill_synthetic(op, x, n, seed)
    ws = dev.Workspace()
    bounds = [n * g // G for g in range(G + 1)]
    totals = torch.zeros(G * sz, dtype=torch.uint8, device="cuda")
    parts = torch.zeros(G * sz, dtype=torch.uint8, device="cuda")
    for g in range(G):
        lo, hi = bounds[g], bounds[g + 1]
        dev.reduce_ordered(op, x.data_ptr() + lo * sz, hi - lo, totals.data_ptr() + g * sz, ws)
        dev.mapreduce(op, x.data_ptr() + lo * sz, hi - lo, parts.data_ptr() + g * sz, ws)
    total = torch.zeros(16, dtype=torch.uint8, device="cuda")
    dev.fold(op, parts, G, total)
    y = dev.empty(op, n, "S")
    carry = torch.zeros(sz, dtype=torch.uint8, device="cuda")
    has = torch.zeros(1, dtype=torch.int32, device="cuda")
    for g in range(G):
        lo, hi = bounds[g], bounds[g + 1]
        dev.fold(op, totals, G, carry, exclusive_upto=g, has_out=has)
        torch.cuda.synchronize()
        cin = carry if int(has.item()) else None
        dev.scan(op, False, x.data_ptr() + lo * sz, y.data_ptr() + lo * sz, hi - lo, ws, carry_in=cin)
    torch.cuda.synchronize()
    del x
    rng = np.random.default_rng(5)
    idx = set(int(v) for v in rng.integers(0, n, size=4096))
    for b in bounds[1:-1]:
        idx.update((b - 1, b, b + 1))
    idx.update((0, 1, n - 1))
    idx = np.array(sorted(idx), dtype=np.int64)
    got_at = y.view(torch.float32)[torch.from_numpy(idx).cuda()].cpu().numpy()
    del y
    bad, worst = orc.check_scan_synthetic_at(op, False, seed, idx.astype(np.uint64), got_at, TOL[op])
    assert bad == 0, f"{bad} of {len(idx)} sampled outputs off, worst err/scale {worst:.3e}"
    got = to_np(total[:4], np.float32)
    _, ex, sc = orc.mapreduce_synthetic(op, n, seed)
    ok, rel = orc.within(op, got, ex, sc, TOL[op])
    assert ok, rel
