"""Per-phase DRAM traffic from an ncu --set full report: sum of dram__bytes_read.sum +
dram__bytes_write.sum over the captured launches whose name matches a substring (one query's
launches of that phase), written into profiles/<round>_traffic.json under a config key.

    python tools/ncu_traffic.py REPORT.ncu-rep CONFIG KERNEL_SUBSTRING [OUT_JSON]
"""
import csv
import io
import json
import os
import subprocess
import sys

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def main():
    rep, cfg, sub = sys.argv[1], sys.argv[2], sys.argv[3]
    out = sys.argv[4] if len(sys.argv) > 4 else os.path.join(
        os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "r02_traffic.json")
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, units = rows[0], rows[1]
    ik, ir, iw, it = (h.index(x) for x in ("Kernel Name", "dram__bytes_read.sum", "dram__bytes_write.sum",
                                          "gpu__time_duration.sum"))
    ih = h.index("lts__t_sector_hit_rate.pct") if "lts__t_sector_hit_rate.pct" in h else None
    hits = []
    launches, rd, wr, ms = [], 0.0, 0.0, 0.0
    for r in rows[2:]:
        if sub not in r[ik]:
            continue
        b_r = float(r[ir]) * UNIT.get(units[ir], 1)
        b_w = float(r[iw]) * UNIT.get(units[iw], 1)
        t = float(r[it]) * {"ns": 1e-6, "us": 1e-3, "ms": 1.0}.get(units[it], 1.0)
        launches.append({"kernel": r[ik].split("(")[0], "dram_read_bytes": b_r, "dram_write_bytes": b_w,
                         "duration_ms_under_ncu": t})
        rd, wr, ms = rd + b_r, wr + b_w, ms + t
        if ih is not None:
            hits.append((float(r[ih]), t))
    data = json.load(open(out)) if os.path.exists(out) else {}
    data[cfg] = {"kernel_match": sub, "launches": launches, "dram_bytes_per_query": rd + wr,
                 "dram_read_bytes": rd, "dram_write_bytes": wr, "source": os.path.basename(rep),
                 "l2_hit_rate_pct": (sum(h * t for h, t in hits) / sum(t for _, t in hits)) if hits else None}
    with open(out, "w") as f:
        json.dump(data, f, indent=1)
    print(cfg, len(launches), "launches", f"{(rd + wr) / 1e6:.1f} MB")


if __name__ == "__main__":
    main()
