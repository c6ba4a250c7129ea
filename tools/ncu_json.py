"""Per-launch DRAM bytes and warp instructions of the step's kernels from an
ncu --set full report, keyed by the C-ABI call that launches them -- what
bench.py reads as ``traffic`` and ``issue`` (profiles/rN_traffic.json,
rN_issue.json).

    python tools/ncu_json.py <report.ncu-rep> <config> <round>
"""
import csv
import io
import json
import subprocess
import sys

CALLS = [("preprocess_fwd_kernel", "sb_preprocess_fwd"), ("count_hist", "sb_bin(count_hist)"),
         ("place_kernel", "sb_bin(place)"), ("blend_fwd_kernel", "sb_blend_fwd"),
         ("ssim_stats", "sb_loss_fused(ssim_stats)"),
         ("ssim_adjoint", "sb_loss_fused(ssim_adjoint)"),
         ("loss_grad", "sb_loss_fused(loss_grad)"), ("blend_bwd_kernel", "sb_blend_bwd_partials"),
         ("gather_short", "sb_gather_adjoints(gather_short)"),
         ("chain_flags", "sb_chain_adam_rows(chain_flags)"),
         ("chain_grad", "sb_chain_adam_rows(chain_grad)"),
         ("adam_list", "sb_chain_adam_rows(adam_list)"),
         ("adam_apply", "sb_chain_adam_rows(adam_apply)")]


def main():
    rep, cfg, rnd = sys.argv[1], int(sys.argv[2]), sys.argv[3]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h = rows[0]
    ki = h.index("Kernel Name")
    cols = {k: h.index(k) for k in ("dram__bytes_read.sum", "dram__bytes_write.sum",
                                    "smsp__inst_executed.sum")}
    units = rows[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    traffic, issue = {}, {}
    for r in rows[2:]:
        name = r[ki]
        call = next((c for k, c in CALLS if k in name), None)
        if call is None or call in traffic:
            continue
        f = lambda k: float(r[cols[k]].replace(",", ""))  # noqa: E731
        traffic[call] = int(f("dram__bytes_read.sum") * scale.get(units[cols["dram__bytes_read.sum"]], 1)
                            + f("dram__bytes_write.sum") * scale.get(units[cols["dram__bytes_write.sum"]], 1))
        issue[call] = int(f("smsp__inst_executed.sum"))
    src = (f"profiles/{rnd}_kernels.md (ncu --set full of tools/step_launches.py on config {cfg}, "
           "one steady-state step")
    json.dump({"config": cfg, "source": src + "; dram__bytes_read.sum + dram__bytes_write.sum per launch)",
               "dram_bytes_per_launch": traffic},
              open(f"profiles/{rnd}_traffic.json", "w"), indent=1)
    json.dump({"config": cfg, "source": src + "; smsp__inst_executed.sum: warp instructions per launch)",
               "warp_inst_per_launch": issue},
              open(f"profiles/{rnd}_issue.json", "w"), indent=1)
    print(json.dumps(traffic, indent=1))


if __name__ == "__main__":
    main()
