#!/usr/bin/env python3
"""Per-source-line warp-stall shares of one kernel from an ncu report
(`ncu -i X --page source --csv --print-source cuda,sass`).

    python tools/ncu_lines.py gpurun_out/x.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    cur, hdr, lines, sass = None, None, [], []
    last = None
    for r in csv.reader(io.StringIO(out)):
        if r and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        stall = r[4]
        if not stall.isdigit():
            continue
        if r[0]:
            last = (cur, r[0], r[1])
            lines.append((int(stall), int(r[7] or 0), last))
        else:
            sass.append((int(stall), r[3].strip(), last))
    tot = sum(s for s, _, _ in lines) or 1
    print(f"total stall samples {tot}")
    for s, inst, (f, ln, src) in sorted(lines, key=lambda x: -x[0])[:top]:
        print(f"{100 * s / tot:5.1f}%  {f}:{ln:>5}  inst={inst:>11}  {src.strip()[:90]}")
    print("\ntop SASS")
    for s, ins, (f, ln, _) in sorted(sass, key=lambda x: -x[0])[:top // 2]:
        print(f"{100 * s / tot:5.1f}%  {f}:{ln:>5}  {ins[:80]}")


if __name__ == "__main__":
    main()
