"""Summarise an `ncu --set full` capture of one train step (bench.py --profile
under `ncu --profile-from-start off`): per-kernel device time, DRAM traffic,
occupancy and issue activity, plus the K2 ray-pass DRAM bytes that bench.py
reports as roofline.traffic (profiles/ncu_k2_traffic.json).

    ncu -i REPORT --page raw --csv > raw.csv
    python profiles/collect.py raw.csv OUT_PREFIX [SOURCE_NOTE [WORKLOAD]]

SOURCE_NOTE (e.g. "profiles/r02/v9 at commit abc1234") and WORKLOAD (the
bench's workload name) are stored in the traffic json: bench.py reports the
traffic only for the workload it was captured on, and names its source.
"""
import csv
import json
import sys

K2 = ("tile_raster", "march_scan", "march_fwd", "march_coop", "rec_tile", "DeviceScan", "shade_fwd", "alpha_bwd", "shade_bwd",
      "shade_geo")
COLS = {
    "time_us": ("gpu__time_duration.sum", 1e-3),
    "dram_read_MB": ("dram__bytes_read.sum", 1e-6),
    "dram_write_MB": ("dram__bytes_write.sum", 1e-6),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1.0),
    "issue_active_pct": ("smsp__issue_active.avg.pct_of_peak_sustained_active", 1.0),
    "threads_per_inst": ("smsp__thread_inst_executed_per_inst_executed.ratio", 1.0),
    "regs": ("launch__registers_per_thread", 1.0),
    "dram_gbs": ("dram__bytes.sum.per_second", 1.0),
    "l2_hit_pct": ("lts__t_sector_hit_rate.pct", 1.0),
    "l1_hit_pct": ("l1tex__t_sector_hit_rate.pct", 1.0),
}
RATE_SCALE = {"Tbyte/s": 1e3, "Gbyte/s": 1.0, "Mbyte/s": 1e-3, "byte/s": 1e-9, "Kbyte/s": 1e-6}
UNIT_SCALE = {"ms": 1e3, "us": 1.0, "usecond": 1.0, "msecond": 1e3, "nsecond": 1e-3, "ns": 1e-3,
              "Gbyte": 1e3, "Mbyte": 1.0, "Kbyte": 1e-3, "byte": 1e-6}


def main(path, out, source=None, workload=None):
    rows = list(csv.reader(open(path)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    res = []
    for d in data:
        r = {"kernel": d[hdr.index("Kernel Name")].split("(")[0].replace("void ", "")}
        for k, (m, _) in COLS.items():
            if m not in hdr:
                continue
            i = hdr.index(m)
            v = float(d[i].replace(",", ""))
            u = units[i]
            if k == "time_us":
                v *= UNIT_SCALE.get(u, 1.0)
            elif k == "dram_gbs":
                v *= RATE_SCALE.get(u, 1.0)
            elif k.startswith("dram"):
                v *= UNIT_SCALE.get(u, 1.0)
            r[k] = v
        res.append(r)
    k2 = [r for r in res if any(s in r["kernel"] for s in K2)]
    k2_bytes = sum((r.get("dram_read_MB", 0) + r.get("dram_write_MB", 0)) * 1e6 for r in k2)
    k2_time = sum(r["time_us"] for r in k2)
    json.dump({"dram_bytes_per_launch": k2_bytes, "source": source, "workload": workload,
               "k2_kernels": [r["kernel"] for r in k2],
               "k2_time_us_serialised": k2_time,
               "note": "K2 = the ray-pass kernels of one train step (incl. CUB sorts); ncu --set full, "
                       "--clock-control none, cold caches per replay"},
              open(out + "_k2_traffic.json", "w"), indent=1)
    with open(out + "_summary.md", "w") as f:
        f.write("| kernel | time (us, serialised) | DRAM read MB | DRAM write MB | DRAM GB/s (% of 6455) | "
                "L2 hit % | L1 hit % | warps active % | issue active % | threads/inst | regs |\n"
                "|---|---|---|---|---|---|---|---|---|---|---|\n")
        for r in res:
            g = r.get('dram_gbs', 0)
            f.write(f"| {r['kernel'][:60]} | {r['time_us']:.1f} | {r.get('dram_read_MB', 0):.1f} | "
                    f"{r.get('dram_write_MB', 0):.1f} | {g:.0f} ({100 * g / 6455.3:.0f} %) | "
                    f"{r.get('l2_hit_pct', 0):.1f} | {r.get('l1_hit_pct', 0):.1f} | "
                    f"{r.get('warps_active_pct', 0):.1f} | "
                    f"{r.get('issue_active_pct', 0):.1f} | {r.get('threads_per_inst', 0):.1f} | "
                    f"{r.get('regs', 0):.0f} |\n")
        f.write(f"\nK2 (ray pass) DRAM traffic per step: {k2_bytes / 1e6:.1f} MB; "
                f"serialised K2 time {k2_time:.0f} us\n")
    print(open(out + "_summary.md").read())


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], *(sys.argv[3:5]))
