"""Hot SASS lines and stall reasons of one kernel in an ncu report.

    python tools/ncu_hot.py <report.ncu-rep> <kernel regex> [top]
"""
import csv
import io
import subprocess
import sys


def main():
    rep, kre = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "-k", "regex:" + kre],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h = rows[0]
    for r in rows[2:3]:
        out = []
        for i, k in enumerate(h):
            if "pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued"):
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                if v > 0:
                    out.append((v, k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        tot = sum(v for v, _ in out)
        print("stalls:", ", ".join(f"{k} {100 * v / tot:.0f}%" for v, k in sorted(out, reverse=True)[:8]))
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + kre,
                          "--print-source", "sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(src)))
    blocks, cur, hdr = [], None, None
    for r in rows:
        if r and r[0] == "Kernel Name":
            cur = []
            blocks.append(cur)
            continue
        if r and r[0] == "Address":
            hdr = r
            continue
        if cur is not None:
            cur.append(r)
    data = blocks[0]
    si = hdr.index("Warp Stall Sampling (All Samples)")
    ei = hdr.index("Instructions Executed")
    f = lambda x: float(x) if x not in ("", "-") else 0.0  # noqa: E731
    tot = sum(f(r[si]) for r in data)
    ex = sum(f(r[ei]) for r in data)
    print(f"samples {tot:.0f}, warp instructions {ex:.0f}, sass lines {len(data)}")
    idx = sorted(range(len(data)), key=lambda i: -f(data[i][si]))[:top]
    for i in sorted(idx):
        r = data[i]
        print(f"{i:5d} {100 * f(r[si]) / tot:5.1f}% {r[ei]:>9s}  {r[1][:90]}")


if __name__ == "__main__":
    main()
