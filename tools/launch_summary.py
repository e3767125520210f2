"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list (per-kernel
totals and shares) as a markdown table. Usage: launch_summary.py launches.csv [title]"""

import csv
import sys


def main(path, title="ncu launch list"):
    rows = []
    with open(path) as fh:
        lines = [l for l in fh if l.startswith('"')]
    rd = csv.reader(lines)
    hdr = next(rd)
    iK, iM, iV = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    iU = hdr.index("Metric Unit") if "Metric Unit" in hdr else None
    for r in rd:
        if r[iM] != "gpu__time_duration.sum":
            continue
        v = float(r[iV].replace(",", ""))
        unit = r[iU] if iU is not None else "ns"
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0}.get(unit, 1e-6)
        rows.append((r[iK].split("(")[0], v * scale))
    agg = {}
    for k, ms in rows:
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += ms
    tot = sum(v[1] for v in agg.values())
    print(f"# {title}\n")
    print(f"total launches: {len(rows)}, summed device time {tot:.1f} ms\n")
    print("| kernel | launches | total ms | avg us | share |\n|---|---:|---:|---:|---:|")
    for k, (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:40]:
        print(f"| `{k}` | {n} | {ms:.2f} | {ms / n * 1e3:.1f} | {100 * ms / tot:.1f}% |")


if __name__ == "__main__":
    main(*sys.argv[1:])
