"""Runs every component kernel of bench.py's composite step twice, in spec
order, for one `ncu --set full` capture (development tool), and summarises the
capture into profiles/<round>/{ncu_full_summary.json,traffic.json}.
    ncu --set full --clock-control none --import-source on \
        -k regex:"scan_lag|scan_smem|mapreduce_kernel|gevm_cols|gemv_kernel" -o /tmp/comp \
        python tools/ncu_components.py run
    ncu -i /tmp/comp.ncu-rep --page raw --csv > gpurun_out/comp_raw.csv
    python tools/ncu_components.py summarize gpurun_out/comp_raw.csv profiles/r02"""
import csv
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def run():
    import torch

    import bench
    from paper_2603_18695_b200 import dev
    specs = bench.component_specs()
    ws = dev.Workspace()
    o16 = torch.empty(16, dtype=torch.uint8, device="cuda")
    A = x = None
    for name, kind, op, incl, n, _ in specs:
        if kind in ("matvec", "vecmat"):
            rows, cols = n
            A = dev.empty(op, rows * cols)
            dev.fill_synthetic(op, A, rows * cols, 5)
            x = dev.empty(op, rows)
            dev.fill_synthetic(op, x, rows, 6)
            y = dev.empty(op, rows, "S")
            for _ in range(2):
                (dev.matvec if kind == "matvec" else dev.vecmat)(op, A, rows, cols, x, y, ws)
            del A, x, y
        else:
            src = dev.empty(op, n)
            dev.fill_synthetic(op, src, n, 3)
            dst = dev.empty(op, n, "S") if kind == "scan" else None
            for _ in range(2):
                if kind == "scan":
                    dev.scan(op, incl, src, dst, n, ws)
                else:
                    dev.mapreduce(op, src, n, o16, ws)
            del src, dst
        torch.cuda.synchronize()
        torch.cuda.empty_cache()


METRICS = {
    "ncu_duration_us": "gpu__time_duration.sum",
    "dram_read": "dram__bytes_read.sum",
    "dram_write": "dram__bytes_write.sum",
    "ncu_dram_pct_of_peak": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "registers": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "achieved_occupancy_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "l2_hit_rate_pct": "lts__t_sector_hit_rate.pct",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1, "msecond": 1e3, "nsecond": 1e-3,
         "us": 1, "ms": 1e3, "ns": 1e-3}


def summarize(raw_csv, dst):
    import bench
    specs = bench.component_specs.__wrapped__() if hasattr(bench.component_specs, "__wrapped__") else None
    rows = list(csv.reader(open(raw_csv)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    if specs is None:
        specs = bench.component_specs()
    assert len(data) == 2 * len(specs), (len(data), len(specs))
    out, traffic = {}, {}
    for i, (name, kind, op, incl, n, byts) in enumerate(specs):
        vals = data[2 * i + 1]  # the second (warm) launch
        d = {"kernel": vals[hdr.index("Kernel Name")][:120]}
        for k, m in METRICS.items():
            if m in hdr:
                j = hdr.index(m)
                d[k] = float(vals[j].replace(",", "")) * SCALE.get(units[j], 1)
        d["dram_bytes_per_launch"] = d.get("dram_read", 0) + d.get("dram_write", 0)
        d["algorithmic_bytes"] = byts
        d["traffic_over_algorithmic"] = round(d["dram_bytes_per_launch"] / byts, 4)
        d["ncu_algorithmic_gbs"] = round(byts / (d["ncu_duration_us"] * 1e-6) / 1e9, 1)
        out[name] = d
        traffic[name] = d["dram_bytes_per_launch"]
    Path(dst).mkdir(parents=True, exist_ok=True)
    (Path(dst) / "ncu_full_summary.json").write_text(json.dumps(out, indent=1) + "\n")
    (Path(dst) / "traffic.json").write_text(json.dumps(traffic, indent=1) + "\n")
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run()
    else:
        summarize(sys.argv[2], sys.argv[3])
