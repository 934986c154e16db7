"""Summarise the ncu --set full CSV exports of tools/gpu_round.sh into
profiles/<round>/ncu_full_summary.json and profiles/traffic.json (development tool).
usage: python tools/ncu_summary.py gpurun_out profiles/r01"""
import csv
import json
import sys
from pathlib import Path

KEYS = {
    "ncu_duration_us": ("gpu__time_duration.sum", 1e-3),  # converted below by unit
    "dram_read": ("dram__bytes_read.sum", None),
    "dram_write": ("dram__bytes_write.sum", None),
    "ncu_dram_pct_of_peak": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", None),
    "registers": ("launch__registers_per_thread", None),
    "grid": ("launch__grid_size", None),
    "block": ("launch__block_size", None),
    "achieved_occupancy_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", None),
    "occupancy_limit_registers": ("launch__occupancy_limit_registers", None),
    "occupancy_limit_shared_mem": ("launch__occupancy_limit_shared_mem", None),
    "l2_hit_rate_pct": ("lts__t_sector_hit_rate.pct", None),
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "us": 1, "ms": 1e3, "ns": 1e-3, "usecond": 1,
         "msecond": 1e3, "nsecond": 1e-3}
ALG = {"mapreduce": 4 * 2**30, "scan": 2 * 4 * 2**28, "gevm": 16384 * 16384 * 4 + 2 * 16384 * 4,
       "gemv": 16384 * 16384 * 4 + 2 * 16384 * 4, "copy": 2 * 2 * 2**30}
TRAFFIC_KEY = {"mapreduce": "mapreduce_f32_sumsq_2^30", "scan": "scan_f32_incl_2^28", "gevm": "gevm_f32_16384^2",
               "gemv": "gemv_f32_16384^2", "copy": "vcopy_2GiB"}


def main(src: str, dst: str) -> None:
    out, traffic = {}, {}
    for k, alg in ALG.items():
        p = Path(src) / f"full_{k}_raw.csv"
        if not p.exists():
            continue
        rows = list(csv.reader(p.open()))
        hdr, units, vals = rows[0], rows[1], rows[2]
        d = {"kernel": vals[hdr.index("Kernel Name")]}
        for name, (metric, _) in KEYS.items():
            if metric in hdr:
                i = hdr.index(metric)
                v = float(vals[i].replace(",", ""))
                d[name] = v * SCALE.get(units[i], 1)
        d["dram_bytes_per_launch"] = d.get("dram_read", 0) + d.get("dram_write", 0)
        d["algorithmic_bytes"] = alg
        d["traffic_over_algorithmic"] = round(d["dram_bytes_per_launch"] / alg, 4)
        d["ncu_algorithmic_gbs"] = round(alg / (d["ncu_duration_us"] * 1e-6) / 1e9, 1)
        out[k] = d
        traffic[TRAFFIC_KEY[k]] = d["dram_bytes_per_launch"]
    Path(dst).mkdir(parents=True, exist_ok=True)
    (Path(dst) / "ncu_full_summary.json").write_text(json.dumps(out, indent=1) + "\n")
    tp = Path(dst).parent / "traffic.json"
    old = json.loads(tp.read_text()) if tp.exists() else {}
    old.update(traffic)
    tp.write_text(json.dumps(old, indent=1) + "\n")
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
