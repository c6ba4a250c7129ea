"""Summarise ncu outputs into profiles/ (committed evidence).

    python tools/ncu_summary.py launches <launches.csv> <steps> > profiles/rN_launches.md
    python tools/ncu_summary.py full <report.ncu-rep> > profiles/rN_kernels.md
"""

import collections
import csv
import io
import subprocess
import sys


def _num(s):
    try:
        return float(s.replace(",", ""))
    except ValueError:
        return None


def launches(path, steps):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ki, mi, vi, ui = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value",
                                              "Metric Unit"))
    idx = hdr.index("ID")
    per = collections.OrderedDict()
    for r in rows[start + 1:]:
        if len(r) <= vi:
            continue
        d = per.setdefault(r[idx], {"name": r[ki]})
        v = _num(r[vi])
        unit = r[ui]
        if r[mi] == "gpu__time_duration.sum":
            scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "us": 1.0,
                     "ms": 1e3}.get(unit, 1.0)
            d["us"] = v * scale
        elif r[mi].startswith("dram__bytes"):
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
            d[r[mi]] = v * scale
    agg = collections.OrderedDict()
    for d in per.values():
        name = d["name"].split("(")[0].replace("void ", "")
        a = agg.setdefault(name, {"n": 0, "us": 0.0, "bytes": 0.0})
        a["n"] += 1
        a["us"] += d.get("us", 0.0)
        a["bytes"] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    total = sum(a["us"] for a in agg.values())
    print(f"# ncu launch list ({len(per)} launches; {steps} steps incl. warm-up/e2e/timing passes)\n")
    print("Cold-cache, serialised per-launch times (`--clock-control none`): compare SHARES.\n")
    print("| kernel | launches | total us | share | avg us | DRAM MB/launch | GB/s |")
    print("|---|---:|---:|---:|---:|---:|---:|")
    for name, a in sorted(agg.items(), key=lambda kv: -kv[1]["us"]):
        avg = a["us"] / a["n"]
        mb = a["bytes"] / a["n"] / 1e6
        gbs = (a["bytes"] / a["n"]) / (avg * 1e-6) / 1e9 if avg > 0 else 0
        print(f"| `{name[:60]}` | {a['n']} | {a['us']:.1f} | {100 * a['us'] / total:.1f}% | "
              f"{avg:.1f} | {mb:.2f} | {gbs:.0f} |")


WANT = [("gpu__time_duration.sum", "duration"),
        ("dram__bytes_read.sum", "DRAM read"),
        ("dram__bytes_write.sum", "DRAM write"),
        ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %peak"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %peak"),
        ("lts__t_sector_hit_rate.pct", "L2 hit %"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
        ("launch__registers_per_thread", "regs"),
        ("smsp__inst_executed.sum", "warp instr"),
        ("lts__t_sectors_op_red.sum", "L2 red sectors"),
        ("lts__t_sectors_op_atom.sum", "L2 atom sectors"),
        ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 %peak")]


def stalls(hdr, r, top=4):
    """Top warp stall reasons (pc sampling) of one kernel row, as % of samples."""
    out = []
    for i, k in enumerate(hdr):
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
            v = _num(r[i])
            if v:
                out.append((v, k[len("smsp__pcsamp_warps_issue_stalled_"):]))
    tot = sum(v for v, _ in out) or 1.0
    return ", ".join(f"{k} {100 * v / tot:.0f}%" for v, k in sorted(out, reverse=True)[:top])


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    print("# ncu --set full: top kernels (one launch each)\n")
    cols = [(m, label) for m, label in WANT if m in hdr]
    print("| kernel | " + " | ".join(label for _, label in cols) + " | top stalls |")
    print("|---|" + "---:|" * len(cols) + "---|")
    seen = set()
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "")
        key = (name, r[hdr.index("ID")] if "ID" in hdr else "")
        if name in seen:
            continue
        seen.add(name)
        vals = []
        for m, _ in cols:
            i = hdr.index(m)
            vals.append(f"{r[i]} {units[i]}".strip())
        print(f"| `{name[:50]}` | " + " | ".join(vals) + f" | {stalls(hdr, r)} |")


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "?")
    else:
        full(sys.argv[2])
