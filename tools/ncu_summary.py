"""Markdown summary of an `ncu --set full` report of the apply kernels: per launch the duration,
DRAM bytes against the SURVEY.md 8(d) algorithmic bytes, FP64 / shared / issue activity,
registers, warps and the top stall reasons.
Usage: python tools/ncu_summary.py report.ncu-rep n_side [pass names in launch order]"""
import csv
import io
import os
import re
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402

rep, n = sys.argv[1], int(sys.argv[2])
names = sys.argv[3:] or ["A_fwd_x", "B_fwd_y", "C_fwd_z_mul_inv_z", "D_inv_y", "E_inv_x_crop"]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]


def val(row, key, scale=1.0):
    i = hdr.index(key)
    u = units[i]
    v = float(row[i].replace(",", ""))
    mult = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "Tbyte": 1e12}.get(u, 1.0)
    if u in ("ms",):
        return v
    if u in ("us", "usecond"):
        return v / 1e3
    if u in ("ns", "nsecond"):
        return v / 1e6
    return v * mult * scale


P = tuple(bench.fus_padded(n)) if hasattr(bench, "fus_padded") else None
if P is None:
    from paper_2011_03009_b200 import fus

    cfg = bench.CFG2 if n == 256 else dict(bench.CFG5, n=n)
    h, _, _ = bench.geometry(cfg)
    g = fus.make_grid([0, 0, 0], [n * h] * 3, h, cfg["harmonic"])
    P = fus.padded_dims(g)
    dims = g.dims
per, _ = bench.algorithmic_bytes(dims, P)
peak, _ = bench.peaks()
stall_cols = [i for i, h in enumerate(hdr) if re.match(r"smsp__average_warps_issue_stalled_.*_per_issue_active\.ratio$", h)]
print(f"grid {tuple(dims)}, padded {tuple(P)}; HBM peak {peak} GB/s (MEASURED_PEAKS.json)\n")
print("| Pass | Kernel | ms | DRAM read GB | DRAM write GB | alg GB | traffic/alg | HBM frac | FP64 pipe % | "
      "issue % | regs | warps/SM | top stalls (per issue) |")
print("|---|---|---|---|---|---|---|---|---|---|---|---|---|")
for name, row in zip(names, data):
    ms = val(row, "gpu__time_duration.sum")
    rd, wr = val(row, "dram__bytes_read.sum") / 1e9, val(row, "dram__bytes_write.sum") / 1e9
    alg = per[name] / 1e9
    fp64 = float(row[hdr.index("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active")])
    issue = float(row[hdr.index("smsp__issue_active.avg.pct_of_peak_sustained_active")])
    regs = row[hdr.index("launch__registers_per_thread")]
    warps = float(row[hdr.index("sm__warps_active.avg.per_cycle_active")])
    st = sorted(((float(row[i] or 0), hdr[i].replace("smsp__average_warps_issue_stalled_", "")
                  .replace("_per_issue_active.ratio", "")) for i in stall_cols), reverse=True)
    st = ", ".join(f"{s} {v:.2f}" for v, s in st if s not in ("selected",))[:60]
    kern = row[hdr.index("Kernel Name")].split("(")[0].replace("void ", "")
    print(f"| {name} | `{kern}` | {ms:.2f} | {rd:.2f} | {wr:.2f} | {alg:.2f} | {(rd + wr) / alg:.3f} | "
          f"{alg / ms / 1e-3 / peak:.3f} | {fp64:.1f} | {issue:.1f} | {regs} | {warps:.1f} | {st} |")
