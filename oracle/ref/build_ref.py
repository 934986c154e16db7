#!/usr/bin/env python3
"""Recipe: compile the reference CPU VM from /root/reference into oracle/_ref/.

ORACLE BUILD SUPPORT ONLY.  Nothing here is product code.

The reference does not build as shipped:
  * bitstype.hpp:27-30 declares `struct Field { TypeDescriptor type; ... }`
    inside the still-incomplete TypeDescriptor (GCC 13: incomplete type);
  * Boost.Context (proj/CMakeLists.txt:13) is not installed and there is no
    network, so proj/src/fiber.hpp's <boost/context/fiber.hpp> is supplied by
    our own stand-in under oracle/ref/shim/;
  * tests/ and capi.cpp are absent, so CMake is not used: the three translation
    units the primitives need (bitstype.cpp, intrinsics.cpp, machine.cpp) are
    compiled directly (litmus.cpp is out of scope and skipped).

The reference sources are copied into the git-ignored build directory
oracle/_ref/src/ (a build intermediate, never committed), the one-line
bitstype.hpp patch is applied there by exact string replacement, and the
result is linked with oracle/ref/ref_driver.cpp into oracle/_ref/libforge_ref.so.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
ORACLE = HERE.parent
OUT = ORACLE / "_ref"
REF = Path(os.environ.get("FORGE_REFERENCE", "/root/reference")) / "proj"

FIELD_NESTED = """  struct Field {
    TypeDescriptor type;
    uint32_t offset;
  };
"""
FIELD_FWD = "  struct Field;\n"
FIELD_OUT_OF_LINE = """
struct TypeDescriptor::Field {
  TypeDescriptor type;
  uint32_t offset;
};
"""
CLASS_END_ANCHOR = "  std::vector<Field> fields_;  // tuple elements carry computed offsets too\n};\n"


def patch_bitstype(path: Path) -> None:
    text = path.read_text()
    if FIELD_NESTED not in text or CLASS_END_ANCHOR not in text:
        raise SystemExit(f"bitstype.hpp patch anchors not found in {path}")
    text = text.replace(FIELD_NESTED, FIELD_FWD, 1)
    text = text.replace(CLASS_END_ANCHOR, CLASS_END_ANCHOR + FIELD_OUT_OF_LINE, 1)
    path.write_text(text)


def run(cmd: list[str]) -> None:
    print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)


def build(force: bool = False) -> Path:
    lib = OUT / "libforge_ref.so"
    if not REF.exists():
        if lib.exists():
            return lib
        raise SystemExit(f"reference not found at {REF} and no prebuilt {lib}")
    inputs = [HERE / "ref_driver.cpp", HERE / "shim" / "ctx_swap.S",
              HERE / "shim" / "boost" / "context" / "fiber.hpp", Path(__file__)]
    if lib.exists() and not force:
        newest = max(p.stat().st_mtime for p in inputs)
        if lib.stat().st_mtime >= newest:
            return lib
    src = OUT / "src"
    if src.exists():
        shutil.rmtree(src)
    src.mkdir(parents=True)
    shutil.copytree(REF / "include", src / "include")
    shutil.copytree(REF / "src", src / "src")
    for p in src.rglob("*"):
        if p.is_file():
            p.chmod(0o644)
    patch_bitstype(src / "include" / "forge" / "bitstype.hpp")

    obj = OUT / "obj"
    obj.mkdir(exist_ok=True)
    flags = ["-std=c++20", "-O2", "-fPIC", "-pthread", "-w",
             f"-I{src / 'include'}", f"-I{HERE / 'shim'}"]
    objs = []
    for tu in ("bitstype.cpp", "intrinsics.cpp", "machine.cpp"):
        o = obj / (tu + ".o")
        run(["g++", *flags, "-c", str(src / "src" / tu), "-o", str(o)])
        objs.append(str(o))
    o = obj / "ctx_swap.o"
    run(["gcc", "-c", str(HERE / "shim" / "ctx_swap.S"), "-o", str(o)])
    objs.append(str(o))
    o = obj / "ref_driver.o"
    run(["g++", *flags, "-c", str(HERE / "ref_driver.cpp"), "-o", str(o)])
    objs.append(str(o))
    run(["g++", "-shared", "-pthread", "-o", str(lib), *objs])
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv))
