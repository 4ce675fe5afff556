"""Source lines of an ncu --set full report (--import-source, -lineinfo) ranked by
warp-stall samples: share of executed instructions and of samples per line.
usage: python scripts/ncu_hot_lines.py REPORT.ncu-rep [N] [FUNCTION-SUBSTRING]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
fsel = sys.argv[3] if len(sys.argv) > 3 else None
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
cur, hdr, agg, fn = None, None, [], ""
for r in csv.reader(txt.splitlines()):
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if len(r) >= 2 and r[0] == "Function Name":
        fn = r[1]
        continue
    if fsel and fsel not in fn:
        continue
    if len(r) > 2 and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) > 8 and r[0]:
        try:
            line, samples, inst = int(r[0]), int(r[4] or 0), int(r[7] or 0)
        except ValueError:
            continue
        agg.append((samples, inst, cur, line, r[1].strip()[:90]))
ts = sum(a[0] for a in agg) or 1
ti = sum(a[1] for a in agg) or 1
print(f"| stall samples | instructions | line | source |\n|---|---|---|---|")
for s, i, f, l, src in sorted(agg, reverse=True)[:top]:
    print(f"| {100 * s / ts:.1f}% | {100 * i / ti:.1f}% | {f}:{l} | `{src.replace('|', '/')}` |")
