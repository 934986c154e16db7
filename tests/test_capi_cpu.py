"""C-ABI checks that need no GPU: libforge.so loads, exports every symbol
include/forge.h declares, serves the host-only calls, and fails LOUDLY (status
NoDevice, never a silent CPU result) when no device is present."""
from __future__ import annotations

import ctypes as C
import re
from pathlib import Path

import pytest

from paper_2603_18695_b200 import capi
from paper_2603_18695_b200 import forge as F

HEADER = Path(__file__).resolve().parents[1] / "include" / "forge.h"


def declared_functions() -> set[str]:
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return set(re.findall(r"\b(forge_[a-z0-9_]+)\s*\(", text))


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(str(capi.LIB_PATH))
    decl = declared_functions()
    assert len(decl) >= 40
    missing = [s for s in sorted(decl) if not hasattr(lib, s)]
    assert not missing, f"libforge.so lacks {missing}"
    # the ctypes binding declares exactly the header's surface
    assert set(capi.exported_symbols()) == decl


def test_abi_version_and_op_menu():
    lib = capi.load()
    assert lib.forge_abi_version() == 1
    info = F.op_info(capi.AFFINE_F32)
    assert info == {"t_size": 8, "s_size": 8, "commutative": False, "binary": False, "name": "affine_f32"}
    assert F.op_info(capi.UF8_F32_SUM)["t_size"] == 1 and F.op_info(capi.UF8_F32_SUM)["s_size"] == 4
    assert F.op_info(capi.MV_MAT2_U32)["binary"] is True
    for op in capi.OPS_1D + capi.OPS_2D:
        assert F.op_info(op)["t_size"] == F.t_dtype(op).itemsize
        assert F.op_info(op)["s_size"] == F.s_dtype(op).itemsize
    with pytest.raises(F.ForgeError):
        F.op_info(99)


def test_vload_pattern_kats():
    assert F.vload_pattern(0, 4) == [4]
    assert F.vload_pattern(1, 4) == [1, 2, 1]
    assert F.vload_pattern(2, 4) == [2, 2]
    assert F.vload_pattern(3, 8) == [1, 4, 2, 1]
    with pytest.raises(F.ForgeError) as e:
        F.vload_pattern(0, 3)
    assert e.value.name == "InvalidNitem"


def test_descriptor_literals():
    assert F.descriptor_info("f32") == (4, 4, "f32")
    assert F.descriptor_info("tuple(u8, f64)") == (16, 8, "tuple(u8,f64)")
    assert F.descriptor_info("struct(u8@0,f64@8,u16@16; size=24)") == (24, 8, "struct(u8@0,f64@8,u16@16;size=24)")
    assert F.descriptor_info("tuple(f32,tuple(u16,u16))")[0] == 8
    for bad, name in (("f16", "ParseError"), ("tuple(", "ParseError"), ("struct(u32@2;size=8)", "InvalidDescriptor"),
                      ("struct(f64@0;size=4)", "InvalidDescriptor"), ("f32 x", "ParseError")):
        with pytest.raises(F.ForgeError) as e:
            F.descriptor_info(bad)
        assert e.value.name == name, bad
    a = bytes([1, 9, 9, 9, 9, 9, 9, 9]) + bytes(8) + bytes([2, 0]) + bytes([7] * 6)
    b = bytes([1, 0, 0, 0, 0, 0, 0, 0]) + bytes(8) + bytes([2, 0]) + bytes([0] * 6)
    assert F.value_bytes_equal("struct(u8@0,f64@8,u16@16;size=24)", a, b)  # padding-blind
    assert not F.value_bytes_equal("tuple(u8,f64,u16)", a[:0] + bytes([3]) + a[1:], b)


def test_arch_params_defaults_and_workspace_sizing():
    p = F.ArchParams()
    assert (p.warp_width, p.mapreduce_blocks, p.threads_per_block, p.nitem_scan) == (32, 100, 256, 16)
    # B200 workspace sizes: 256-byte control block + one 256-byte slot per
    # 32-byte group of two 16-byte tile states (the f64 carry of an f32 sum) —
    # two 8192-f32 tiles of the smem kernel (full speed); never less than the
    # general kernel's 4096-element tiles at packed 16-byte states
    assert F.required_workspace(capi.PRIM_SCAN, 4, 4096) == 256 + 256
    assert F.required_workspace(capi.PRIM_SCAN, 4, 8192) == 256 + 256
    assert F.required_workspace(capi.PRIM_SCAN, 4, 16384) == 256 + 256
    assert F.required_workspace(capi.PRIM_SCAN, 4, 16385) == 256 + 512
    assert F.required_workspace(capi.PRIM_SCAN, 4, 1 << 33) == 256 + (1 << 19) * 256
    assert F.required_workspace(capi.PRIM_VCOPY, 4, 100) == 0
    # the reference-facing bound covers the device layer's need for every menu op
    # (a workspace made for S fits every T: ADVICE r01)
    lib = capi.load()
    for op in capi.OPS_1D:
        ss = F.op_info(op)["s_size"]
        for n in (1, 4095, 4097, 100_003, 1 << 24):
            need = C.c_uint64()
            assert lib.forge_dev_workspace_bytes(capi.PRIM_SCAN, op, n, 0, C.byref(need)) == 0
            assert F.required_workspace(capi.PRIM_SCAN, ss, n) >= need.value, (op, n)
    with pytest.raises(F.ForgeError) as e:
        F.required_workspace(capi.PRIM_SCAN, 4, 10, params=F.ArchParams(warp_width=64, threads_per_block=256))
    assert e.value.name == "Unsupported"
    with pytest.raises(F.ForgeError) as e:
        F.required_workspace(capi.PRIM_SCAN, 4, 10, params=F.ArchParams(warp_width=48))
    assert e.value.name == "InvalidArgument"
    with pytest.raises(F.ForgeError) as e:
        F.required_workspace(capi.PRIM_SCAN, 4, 10, params=F.ArchParams(nitem_scan=3))
    assert e.value.name == "InvalidNitem"


def test_no_device_fails_loudly():
    if F.device_count() > 0:
        pytest.skip("a GPU is present")
    with pytest.raises(F.ForgeError) as e:
        F.Machine(0)
    assert e.value.name == "NoDevice"
    lib = capi.load()
    ws = C.c_uint64()
    rc = lib.forge_dev_workspace_bytes(capi.PRIM_SCAN, capi.F32_SUM, 1000, 0, C.byref(ws))
    assert rc == 0 and ws.value > 256   # pure host arithmetic works


def test_shard_ranges_and_group_without_device():
    # forge_shard_range is host arithmetic (shard r = [total*r/G, total*(r+1)/G))
    from paper_2603_18695_b200 import group
    for total in (0, 1, 3, 10, 1 << 33, (1 << 64) - 1):
        for G in (1, 2, 3, 8):
            spans = [group.shard_range(total, r, G) for r in range(G)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(spans[i][1] == spans[i + 1][0] for i in range(G - 1))
            assert max(h - l for l, h in spans) - min(h - l for l, h in spans) <= 1
    with pytest.raises(F.ForgeError):
        group.shard_range(10, 3, 3)
    lib = capi.load()
    n = C.c_int()
    lib.forge_device_count(C.byref(n))
    if n.value == 0:  # this container: no device, no fallback
        h = C.c_void_p()
        devs = (C.c_int32 * 2)(0, 0)
        assert lib.forge_group_create(devs, 2, C.byref(h)) == capi.ERR_NO_DEVICE
