"""profiles/r2_rayleigh_fp64.json from an ncu metrics run of the Rayleigh grid kernel:
ncu --metrics sm__inst_executed_pipe_fp64.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,
smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,
smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second
--csv --clock-control none -k regex:monopole_grid -c 1 python tools/profile_monopole.py 1 > ncu.csv
Usage: python tools/rayleigh_fp64.py ncu.csv"""
import csv
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if l.startswith('"'))]
hdr = rows[0]
m = {}
name = None
for r in rows[1:]:
    m[r[hdr.index("Metric Name")]] = (float(r[hdr.index("Metric Value")].replace(",", "")), r[hdr.index("Metric Unit")])
    name = r[hdr.index("Kernel Name")]
terms = 301 * 323 * 323 * 4096  # cfg4-desk D2 grid x 4096 sources (tools/profile_monopole.py)
warp = m["sm__inst_executed_pipe_fp64.sum"][0]
t_ms = m["gpu__time_duration.sum"][0] * {"ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}[m["gpu__time_duration.sum"][1]]
out = {
    "_source": "ncu --metrics sm__inst_executed_pipe_fp64.sum,sm__pipe_fp64_cycles_active,smsp__sass_thread_inst_executed_op_{dfma,dadd,dmul}_pred_on.sum --clock-control none -k regex:monopole_grid -c 1 python tools/profile_monopole.py 1 (cfg4-desk D2 grid 301x323x323, 4096 sources) on one B200, round 2 (ring-reused x part); tools/rayleigh_fp64.py",
    "kernel": name,
    "terms": terms,
    "kernel_ms": t_ms,
    "fp64_warp_instr": warp,
    "fp64_thread_instr_per_term": warp * 32 / terms,
    "dfma_dadd_dmul_thread_instr": [m[f"smsp__sass_thread_inst_executed_op_{o}_pred_on.sum"][0] for o in ("dfma", "dadd", "dmul")],
    "fp64_pipe_pct_ncu": m["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"][0],
    "sm_clock_hz": m["sm__cycles_elapsed.avg.per_second"][0] * {"hz": 1.0, "khz": 1e3, "mhz": 1e6, "ghz": 1e9}[m["sm__cycles_elapsed.avg.per_second"][1].lower()],
    "terms_per_s_ncu": terms / (t_ms * 1e-3),
}
json.dump(out, open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "r2_rayleigh_fp64.json"), "w"), indent=1)
print(json.dumps(out, indent=1))
