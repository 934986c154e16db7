"""SASS evidence for the product kernels (cuobjdump -sass of the built
libforge.so): per kernel family, one representative instantiation's
instruction-mnemonic histogram of the memory/sync instructions that prove the
Blackwell-native paths (UTMALDG/UTMASTG = TMA, SYNCS = mbarrier, LDG...256 =
256-bit loads, IDP4A, ...) plus a short excerpt.  Writes profiles/<round>/sass/.
    python tools/sass_excerpts.py r02"""
import collections
import json
import re
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
out_dir = ROOT / "profiles" / (sys.argv[1] if len(sys.argv) > 1 else "r02") / "sass"
out_dir.mkdir(parents=True, exist_ok=True)
lib = ROOT / "paper_2603_18695_b200" / "libforge.so"
sass = subprocess.run(["cuobjdump", "-sass", str(lib)], capture_output=True, text=True, check=True).stdout
funcs = re.split(r"\n\s+Function : ", sass)
# family -> substring of the mangled name that picks one representative
FAMILIES = {
    "scan_lag_kernel (affine, f64 carry)": ("scan_lag_kernel", "AffineOpELb1"),
    "scan_smem_kernel (Mat2, 16-byte elements, R = 2)": ("scan_smem_kernel", "Mat2MulELb1ELi2"),
    "scan_smem_kernel (f32 sum, TMA tile)": ("scan_smem_kernel", "IffNS_3alg8IdentityENS_4menu6AddF32ELb1"),
    "scan_smem_kernel (affine, f64 carry)": ("scan_smem_kernel", "AffineOpELb1"),
    "scan_smem_kernel (argmax)": ("scan_smem_kernel", "ArgMaxOpELb1"),
    "mapreduce_kernel (f32 sum-of-squares)": ("mapreduce_kernel", "IffNS_3alg6SquareENS_4menu6AddF32"),
    "mapreduce_kernel (i32 max)": ("mapreduce_kernel", "IiiNS_3alg8IdentityENS_4menu6MaxI32"),
    "code_sum_kernel (UnitFloat8 exact sum)": ("code_sum_kernel", ""),
    "gevm_cols_kernel (f32 plus-times)": ("gevm_cols_kernel", "IffNS_4menu6MulF32ENS2_6AddF32"),
    "gemv_kernel (f32 plus-times)": ("gemv_kernel", "IffNS_4menu6MulF32ENS2_6AddF32"),
    "vcopy_kernel": ("vcopy_kernel", ""),
    "reduce_ordered_kernel (f32 sum)": ("reduce_ordered_kernel", "IffNS_3alg8IdentityENS_4menu6AddF32"),
}
KEYS = ["UTMALDG", "UTMASTG", "UTMAPF", "UBLKCP", "SYNCS", "LDG.E.NA.ENL2.256", "LDG.E.ENL2.256", "LDG", "STG", "LDS", "STS",
        "IDP.4A", "ATOMG", "RED", "CCTL", "FENCE", "SHFL", "DFMA", "DMUL", "DADD", "FFMA", "FADD", "FMNMX", "MEMBAR", "ERRBAR"]
summary = {}
for fam, (kname, sub) in FAMILIES.items():
    cands = [f for f in funcs if f.split("\n", 1)[0].find(kname) >= 0 and sub in f.split("\n", 1)[0]]
    if not cands:
        summary[fam] = {"missing": True}
        continue
    f = cands[0]
    name = f.split("\n", 1)[0].strip()
    ins = re.findall(r"/\*[0-9a-f]{4,}\*/\s+([^;]+);", f)
    ops = [i.split()[0] if not i.startswith("@") else i.split()[1] for i in ins]
    hist = collections.Counter()
    for o in ops:
        for k in KEYS:
            if o.startswith(k):
                hist[k] += 1
                break
    summary[fam] = {"mangled": name[:160], "instructions": len(ins), "memory_sync_histogram": dict(hist)}
    keep = [i.strip() for i in ins if re.match(r"(@\S+\s+)?(UTMA|SYNCS|LDG|STG|IDP|ATOMG|FENCE|UBLKCP)", i.strip())]
    (out_dir / (re.sub(r"[^a-z0-9]+", "_", fam.lower()).strip("_") + ".sass.txt")).write_text(
        f"// {fam}\n// {name}\n// memory / sync instructions in program order (first 80)\n" + "\n".join(keep[:80]) + "\n")
(out_dir / "summary.json").write_text(json.dumps(summary, indent=1) + "\n")
print(json.dumps({k: v.get("memory_sync_histogram") for k, v in summary.items()}, indent=1))
