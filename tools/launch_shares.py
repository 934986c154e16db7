"""Kernel shares of the headline step from an ncu launch list of
`bench.py --steps S --warmup W` (development tool): the product-kernel
launches of the S timed steps (after W warm-up steps of the same 8 launches),
their per-family ncu times (cold-cache, serialised: compare shares, not
absolutes) and shares of the step.
    python tools/launch_shares.py gpurun_out/launches.csv 2 3 > profiles/r02/launch_shares_step.json"""
import collections
import csv
import json
import sys

path, steps, warm = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
FAM = ["scan_smem_kernel", "scan_lag_kernel", "mapreduce_kernel", "code_sum_kernel", "gevm_cols_kernel",
       "gevm_kernel", "gemv_kernel", "reduce_ordered_kernel", "fold_kernel"]
rows = [r for r in csv.reader(open(path)) if len(r) > 14 and r[0] != "ID"]
prod = []
for r in rows:
    name = r[4]
    fam = next((f for f in FAM if f in name), None)
    if fam and r[12] == "gpu__time_duration.sum":
        prod.append((fam, float(r[14].replace(",", "")) * (1e-3 if r[13] == "ns" else 1.0), r[8]))
PER_STEP = 8
timed = prod[warm * PER_STEP:(warm + steps) * PER_STEP]
tot = collections.defaultdict(float)
for fam, us, grid in timed:
    tot[fam] += us
step_us = sum(tot.values()) / steps
out = {"launches_per_step": PER_STEP, "steps": steps, "ncu_step_us": round(step_us, 1),
       "families": {f: {"us_per_step": round(v / steps, 1), "share": round(v / steps / step_us, 4)}
                    for f, v in sorted(tot.items(), key=lambda kv: -kv[1])},
       "launch_order": [(f, round(us, 1), g) for f, us, g in timed[:PER_STEP]]}
print(json.dumps(out, indent=1))
