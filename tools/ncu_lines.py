"""Summarise an ncu report per CUDA source line (stall samples, instructions).

    python tools/ncu_lines.py report.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    by = 1 if len(sys.argv) > 3 and sys.argv[3] == "inst" else 0
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    cur = None
    hdr = None
    agg = {}
    for r in rows:
        if len(r) >= 2 and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr) or not r[0].isdigit():
            continue
        st = float(r[4] or 0) if r[4] not in ("-", "") else 0.0
        ins = float(r[7] or 0) if r[7] not in ("-", "") else 0.0
        key = (cur, int(r[0]))
        a = agg.setdefault(key, [0.0, 0.0, r[1][:100]])
        a[0] += st
        a[1] += ins
    ts = sum(v[0] for v in agg.values()) or 1
    ti = sum(v[1] for v in agg.values()) or 1
    print(f"total stall samples {ts:.0f}, instructions {ti:.3e}")
    for (f, ln), (st, ins, src) in sorted(agg.items(), key=lambda kv: -kv[1][by])[:top]:
        print(f"{st / ts * 100:5.1f}% {ins / ti * 100:5.1f}%  {f}:{ln:<4d} {src}")


if __name__ == "__main__":
    main()
