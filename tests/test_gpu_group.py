"""Native single-process multi-GPU layer (include/forge.h forge_group_* /
forge_sharded_*, csrc/group.cu) against the CPU oracle, SURVEY.md §8(e).

On a 1-GPU box: G = 1 runs the NCCL path (a one-device ncclCommInitAll clique);
G = 2 and 4 run the EMULATED group (every shard on cuda:0, the same exchange
logic, the all-gather by device copies), including empty shards."""
from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle as orc
from tests.helpers import assert_match

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
capi = pytest.importorskip("paper_2603_18695_b200.capi")
group = pytest.importorskip("paper_2603_18695_b200.group")
F = pytest.importorskip("paper_2603_18695_b200.forge")

GROUPS = [[0], [0, 0], [0, 0, 0, 0]]


@pytest.fixture(scope="module", params=GROUPS, ids=lambda d: f"G{len(d)}")
def grp(request):
    g = group.Group(request.param)
    yield g
    g.close()


def dev_bytes(arr: np.ndarray) -> "torch.Tensor":
    b = np.ascontiguousarray(arr).view(np.uint8)
    return torch.from_numpy(b.copy()).cuda() if b.size else torch.empty(0, dtype=torch.uint8, device="cuda")


def split(x: np.ndarray, G: int):
    parts, ns = [], []
    for r in range(G):
        lo, hi = group.shard_range(len(x), r, G)
        parts.append(dev_bytes(x[lo:hi]))
        ns.append(hi - lo)
    return parts, ns


@pytest.mark.parametrize("op", [capi.F32_SUMSQ, capi.I32_MAX, capi.UF8_F32_SUM, capi.ARGMAX_F32I32, capi.I64_SUM])
@pytest.mark.parametrize("n", [3, 100_003, 1 << 22])
def test_group_mapreduce(grp, op, n):
    x = orc.fill(op, n, 0x6A0 + op)
    parts, ns = split(x, grp.size)
    got = np.frombuffer(grp.mapreduce(op, parts, ns), dtype=F.s_dtype(op))
    want, ex, sc = orc.mapreduce(op, x)
    assert_match(op, got, want, ex, sc, f"sharded mapreduce G={grp.size} n={n}")


@pytest.mark.parametrize("op", [capi.MAT2_U32, capi.F32_SUM, capi.AFFINE_F32, capi.I32_SUM, capi.ARGMAX_F32I32])
@pytest.mark.parametrize("n", [3, 4097, 1_000_003])
@pytest.mark.parametrize("inclusive", [True, False])
def test_group_scan(grp, op, n, inclusive):
    x = orc.fill(op, n, 0x6B0 + op)
    parts, ns = split(x, grp.size)
    ss = F.s_dtype(op).itemsize
    outs = [torch.empty(k * ss, dtype=torch.uint8, device="cuda") for k in ns]
    grp.scan(op, inclusive, parts, outs, ns)
    got = np.concatenate([o.cpu().numpy() for o in outs]).view(F.s_dtype(op))
    want, ex, sc = orc.scan(op, inclusive, x)
    assert_match(op, got, want, ex, sc, f"sharded scan G={grp.size} n={n}")


@pytest.mark.parametrize("op", [capi.MV_F32_PLUS_TIMES, capi.MV_F32_MIN_PLUS, capi.MV_MAT2_U32])
@pytest.mark.parametrize("shape", [(513, 67), (1000, 3), (2048, 2048)])
def test_group_matvec_vecmat(grp, op, shape):
    n, p = shape
    G = grp.size
    A = orc.fill(op, n * p, 0x6C0 + op)  # column-major n x p
    ss = F.s_dtype(op).itemsize
    # gevm: column blocks (contiguous in column-major)
    x = orc.fill(op, n, 0x6C1 + op)
    blocks, ys, xs = [], [], []
    for r in range(G):
        lo, hi = group.shard_range(p, r, G)
        blocks.append(dev_bytes(A[lo * n: hi * n]))
        ys.append(torch.empty(max(hi - lo, 1) * ss, dtype=torch.uint8, device="cuda"))
        xs.append(dev_bytes(x))
    grp.matvec(op, blocks, n, p, xs, ys)
    got = np.concatenate([ys[r].cpu().numpy()[: (group.shard_range(p, r, G)[1] - group.shard_range(p, r, G)[0]) * ss]
                          for r in range(G)]).view(F.s_dtype(op))
    want, ex, sc = orc.matvec(op, A, n, p, x)
    assert_match(op, got, want, ex, sc, f"sharded matvec G={G} {shape}")
    # gemv: row blocks, each column-major with lda = its row count
    xv = orc.fill(op, p, 0x6C2 + op)
    cols = A.reshape(p, n)  # row j = column j of A
    blocks, zs, xs = [], [], []
    for r in range(G):
        lo, hi = group.shard_range(n, r, G)
        blocks.append(dev_bytes(np.ascontiguousarray(cols[:, lo:hi]).reshape(-1)))
        zs.append(torch.empty(max(hi - lo, 1) * ss, dtype=torch.uint8, device="cuda"))
        xs.append(dev_bytes(xv))
    grp.vecmat(op, blocks, n, p, xs, zs)
    got = np.concatenate([zs[r].cpu().numpy()[: (group.shard_range(n, r, G)[1] - group.shard_range(n, r, G)[0]) * ss]
                          for r in range(G)]).view(F.s_dtype(op))
    want, ex, sc = orc.vecmat(op, A, n, p, xv)
    assert_match(op, got, want, ex, sc, f"sharded vecmat G={G} {shape}")


def test_group_errors():
    with pytest.raises(F.ForgeError) as e:
        group.Group([])
    assert e.value.status == capi.ERR_INVALID_ARGUMENT
    with pytest.raises(F.ForgeError):
        group.Group([0, 99])


# ---- block-cyclic shards + cross-GPU decoupled look-back (forge_sharded_scan_cyclic)

@pytest.mark.parametrize("op", [capi.I32_SUM, capi.ARGMAX_F32I32, capi.F32_SUM, capi.AFFINE_F32])
@pytest.mark.parametrize("inclusive", [True, False])
def test_group_scan_cyclic(grp, op, inclusive):
    q = group.cyclic_quantum(op)
    G = grp.size
    tpc = max(1, min(16, 148 // G))           # chunk tiles: the emulated group needs tpc * G <= SMs
    chunk = tpc * q
    for n in (5, chunk - 3, 3 * chunk + 17, (4 * G + 1) * chunk + q // 2 + 1, 64 * chunk):
        x = orc.fill(op, n, 0x6D0 + op + n)
        spans = group.cyclic_split(n, chunk, G)
        ss = F.s_dtype(op).itemsize
        src, dst = [], []
        for r in range(G):
            local = np.concatenate([x[lo:hi] for lo, hi in spans[r]]) if spans[r] else x[:0]
            assert len(local) == group.cyclic_local_n(n, chunk, r, G)
            src.append(dev_bytes(local))
            dst.append(torch.empty(max(len(local), 1) * ss, dtype=torch.uint8, device="cuda"))
        grp.scan_cyclic(op, inclusive, src, dst, n, chunk)
        got = np.empty(n, dtype=F.s_dtype(op))
        for r in range(G):
            loc = dst[r].cpu().numpy().view(F.s_dtype(op))
            off = 0
            for lo, hi in spans[r]:
                got[lo:hi] = loc[off: off + hi - lo]
                off += hi - lo
        want, ex, sc = orc.scan(op, inclusive, x)
        assert_match(op, got, want, ex, sc, f"cyclic scan G={G} n={n} chunk={chunk}")


def test_group_scan_cyclic_relaunch_bitexact(grp):
    # the relaunch stress of the single-pass protocol, across shards: one
    # workspace set, two inputs alternating, every output bit-exact
    op, G = capi.I32_SUM, grp.size
    q = group.cyclic_quantum(op)
    chunk = max(1, min(16, 148 // G)) * q
    n = 40 * chunk + 1234
    spans = group.cyclic_split(n, chunk, G)
    ins, wants = [], []
    for k in range(2):
        x = orc.fill(op, n, 0x6E0 + k)
        ins.append([dev_bytes(np.concatenate([x[lo:hi] for lo, hi in spans[r]])) for r in range(G)])
        wants.append(orc.scan(op, True, x)[0])
    dst = [torch.empty(group.cyclic_local_n(n, chunk, r, G) * 4, dtype=torch.uint8, device="cuda") for r in range(G)]
    for i in range(12):
        grp.scan_cyclic(op, True, ins[i % 2], dst, n, chunk)
        got = np.empty(n, dtype=np.int32)
        for r in range(G):
            loc = dst[r].cpu().numpy().view(np.int32)
            off = 0
            for lo, hi in spans[r]:
                got[lo:hi] = loc[off: off + hi - lo]
                off += hi - lo
        assert np.array_equal(got, wants[i % 2]), i


def test_group_scan_cyclic_rejects():
    with group.Group([0, 0]) as g:
        x = torch.zeros(64, dtype=torch.uint8, device="cuda")
        with pytest.raises(F.ForgeError):  # 16-byte elements: single-pass protocol only
            g.scan_cyclic(capi.MAT2_U32, True, [x, x], [x, x], 2, group.cyclic_quantum(capi.I32_SUM))
        with pytest.raises(F.ForgeError):  # chunk not a multiple of the tile
            g.scan_cyclic(capi.I32_SUM, True, [x, x], [x, x], 16, 100)
