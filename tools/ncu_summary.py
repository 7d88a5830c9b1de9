#!/usr/bin/env python3
"""Summarise ncu evidence into markdown for profiles/.

    python tools/ncu_summary.py --rep gpurun_out/x.ncu-rep --launches gpurun_out/l.csv \
        --algo-bytes 83968000000 --peak 6552.3 --title "..." > profiles/r1_k_sym_agg.md
"""
import argparse
import collections
import csv
import io
import subprocess

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("lts__t_sector_hit_rate.pct", "L2 sector hit rate %"),
    ("l1tex__t_sector_hit_rate.pct", "L1 sector hit rate %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput % of peak"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("smsp__inst_executed.sum", "warp instructions executed"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep")
    ap.add_argument("--launches")
    ap.add_argument("--algo-bytes", type=float, default=0)
    ap.add_argument("--peak", type=float, default=6552.3)
    ap.add_argument("--title", default="")
    ap.add_argument("--command", default="")
    ap.add_argument("--traffic-json", default="", help="record DRAM bytes/launch under this kernel key "
                    "in profiles/ncu_traffic.json (read by bench.py's roofline.traffic)")
    ap.add_argument("--source", default="", help="the profiles/ summary the traffic number comes from")
    a = ap.parse_args()
    print(f"# {a.title}\n")
    if a.command:
        print(f"Command: `{a.command}`\n")
    if a.rep:
        h, units, data = raw(a.rep)
        for row in data:
            name = row[h.index("Kernel Name")] if "Kernel Name" in h else "?"
            print(f"## ncu --set full: `{name[:100]}`\n")
            print("| metric | value | unit |\n|---|---|---|")
            vals = {}
            for k, label in KEYS:
                if k in h:
                    i = h.index(k)
                    vals[k] = (row[i], units[i])
                    print(f"| {label} (`{k}`) | {row[i]} | {units[i]} |")
            if a.algo_bytes and "gpu__time_duration.sum" in vals:
                t, u = vals["gpu__time_duration.sum"]
                t = float(t.replace(",", "")) * {"ms": 1e-3, "us": 1e-6, "ns": 1e-9, "s": 1}[u.strip()]
                ach = a.algo_bytes / t / 1e9
                print(f"\nAlgorithmic bytes {a.algo_bytes / 1e9:.2f} GB / {t * 1e3:.3f} ms (cold, serialised by ncu) = "
                      f"{ach:.0f} GB/s = {ach / a.peak:.3f} of measured peak {a.peak} GB/s.")
                if "dram__bytes_read.sum" in vals:
                    rd, ru = vals["dram__bytes_read.sum"]
                    wr, wu = vals.get("dram__bytes_write.sum", ("0", ru))
                    scale = {"GB": 1e9, "MB": 1e6, "KB": 1e3, "byte": 1, "Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3}
                    tr = float(rd.replace(",", "")) * scale.get(ru.strip(), 1) + float(wr.replace(",", "")) * scale.get(wu.strip(), 1)
                    print(f"DRAM traffic {tr / 1e9:.2f} GB = {tr / a.algo_bytes:.2f}x the algorithmic bytes.")
                    if a.traffic_json:
                        import json
                        from pathlib import Path
                        tj = Path(__file__).resolve().parent.parent / "profiles" / "ncu_traffic.json"
                        d = json.loads(tj.read_text()) if tj.exists() else {}
                        d[a.traffic_json] = {"dram_bytes": int(tr), "algorithmic_bytes": int(a.algo_bytes),
                                             "ncu_ms": round(t * 1e3, 3), "source": a.source}
                        tj.write_text(json.dumps(d, indent=1) + "\n")
            print()
    if a.launches:
        rows = list(csv.reader(open(a.launches)))
        hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
        h = rows[hi]
        ki, mi, mn = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
        seq = [(r[ki], float(r[mi].replace(",", ""))) for r in rows[hi + 1:]
               if len(r) > mi and r[mn] == "gpu__time_duration.sum"]
        starts = [i for i, (n, _) in enumerate(seq) if "k_coll_keys" in n]
        win = seq[starts[-1]:] if starts else seq
        agg = collections.defaultdict(lambda: [0, 0.0])
        for n, v in win:
            agg[n][0] += 1
            agg[n][1] += v
        tot = sum(v for _, v in win)
        print(f"## Launch list (last window: {len(win)} launches, {tot / 1e6:.3f} ms of kernel time; ncu-serialised, "
              f"cold caches — compare shares, not absolutes)\n")
        print("| kernel | launches | ms | share |\n|---|---|---|---|")
        for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1])[:25]:
            print(f"| `{k[:90]}` | {c} | {v / 1e6:.3f} | {100 * v / tot:.1f}% |")


if __name__ == "__main__":
    main()
