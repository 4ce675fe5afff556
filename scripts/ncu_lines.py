"""Per-source-line aggregation of an ncu --page source --print-source cuda,sass CSV export:
top lines by warp-stall samples and by executed instructions."""
import csv
import sys


def rows(path):
    cur = None
    out = []
    with open(path) as fh:
        for r in csv.reader(fh):
            if not r:
                continue
            if r[0] == "File Path":
                cur = r[1].split("/")[-1]
                continue
            if r[0] in ("Function Name", "Line No") or not r[0]:
                continue
            try:
                out.append((cur, int(r[0]), r[1].strip()[:90], int(r[4] or 0), int(r[7] or 0)))
            except (ValueError, IndexError):
                pass
    return out


if __name__ == "__main__":
    rs = rows(sys.argv[1])
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    ts = sum(r[3] for r in rs) or 1
    ti = sum(r[4] for r in rs) or 1
    print(f"total samples {ts}, warp instructions {ti}")
    for r in sorted(rs, key=lambda r: -r[3])[:n]:
        print(f"{100 * r[3] / ts:5.1f}% smp {100 * r[4] / ti:5.1f}% ins  {r[0]}:{r[1]}  {r[2]}")
