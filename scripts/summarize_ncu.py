"""Summaries of ncu captures for profiles/ (launch lists and --set full reports)."""
import collections
import csv
import subprocess
import sys


def launches(path):
    with open(path) as fh:
        lines = [l for l in fh if l.startswith('"')]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        u = r["Metric Unit"]
        v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}.get(u, 1.0)
        name = r["Kernel Name"].split("(")[0].replace("void ", "")
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    out = [f"launch list `{path}` (ncu --metrics gpu__time_duration.sum --clock-control none; cold-cache, serialised)",
           "", f"total {tot / 1e3:.3f} ms over {sum(v[0] for v in agg.values())} launches", "",
           "| kernel | launches | time (ms) | share |", "|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"| `{k}` | {v[0]} | {v[1] / 1e3:.3f} | {100 * v[1] / tot:.1f}% |")
    return "\n".join(out)


WANT = ["Duration", "Executed Ipc Active", "Issue Slots Busy", "L1/TEX Hit Rate", "L2 Hit Rate", "Achieved Occupancy",
        "Registers Per Thread", "Warp Cycles Per Issued Instruction", "Executed Instructions", "DRAM Throughput",
        "Memory Throughput", "Compute (SM) Throughput", "Avg. Active Threads Per Warp"]


def full(path):
    det = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    out = [f"ncu --set full report `{path}`", ""]
    rows = list(csv.reader(det.splitlines()))
    hdr = rows[0]
    per = collections.OrderedDict()
    for row in rows[1:]:
        d = dict(zip(hdr, row))
        if d.get("Metric Name") in WANT:
            key = (d.get("ID"), d["Kernel Name"].split("(")[0])
            per.setdefault(key, {})[d["Metric Name"]] = f'{d["Metric Value"]} {d["Metric Unit"]}'.strip()
    rr = list(csv.reader(raw.splitlines()))
    rh = rr[0]
    traffic = {}
    for row in rr[2:]:
        d = dict(zip(rh, row))
        try:
            rb = float(d.get("dram__bytes_read.sum", "0").replace(",", ""))
            wb = float(d.get("dram__bytes_write.sum", "0").replace(",", ""))
        except ValueError:
            continue
        unit_r, unit_w = rr[1][rh.index("dram__bytes_read.sum")], rr[1][rh.index("dram__bytes_write.sum")]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        traffic[d["ID"]] = rb * scale.get(unit_r, 1) + wb * scale.get(unit_w, 1)
        stalls = sorted(((float(d[k].replace(",", "") or 0), k) for k in rh
                         if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")
                         and d.get(k)), reverse=True)[:6]
        per_key = [k for k in per if k[0] == d["ID"]]
        if per_key:
            per[per_key[0]]["top stalls"] = ", ".join(
                f'{k.replace("smsp__pcsamp_warps_issue_stalled_", "")}={int(v)}' for v, k in stalls)
    for (kid, name), m in per.items():
        out.append(f"### `{name}` (launch id {kid})")
        out.append("")
        for k, v in m.items():
            out.append(f"- {k}: {v}")
        if kid in traffic:
            out.append(f"- DRAM traffic (read + write): {traffic[kid] / 1e6:.1f} MB")
        out.append("")
    return "\n".join(out)


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(launches(p) if p.endswith(".csv") else full(p))
        print()
