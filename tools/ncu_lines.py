"""Stall samples and executed warp instructions per CUDA source line of one
kernel in an ncu report (needs -lineinfo and --import-source on).

    python tools/ncu_lines.py <report.ncu-rep> <kernel regex> [top]
"""
import csv
import io
import subprocess
import sys


def main():
    rep, kre = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + kre,
                          "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, lines, path = None, [], ""
    for r in rows:
        if r and r[0] == "File Path":
            path = r[1].rsplit("/", 1)[-1]
        elif r and r[0] == "Line No":
            hdr = r
        elif hdr and r and r[0] not in ("", "Function Name") and len(r) == len(hdr):
            lines.append((path, r))
    si = hdr.index("Warp Stall Sampling (All Samples)")
    ei = hdr.index("Instructions Executed")
    def f(x):
        try:
            return float(x)
        except ValueError:
            return 0.0
    tot = sum(f(r[si]) for _, r in lines) or 1.0
    ins = sum(f(r[ei]) for _, r in lines) or 1.0
    print(f"samples {tot:.0f}, warp instructions {ins:.0f}")
    for p, r in sorted(lines, key=lambda x: -f(x[1][si]))[:top]:
        print(f"{100 * f(r[si]) / tot:5.1f}% smp {100 * f(r[ei]) / ins:5.1f}% ins  "
              f"{p}:{r[0]:>4s}  {r[1].strip()[:90]}")


if __name__ == "__main__":
    main()
