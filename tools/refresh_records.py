"""Refresh the tracked records from one gpurun_out/<prefix>_* set (the final-validation command in
profiles/README.md): traffic.json and r2_apply_fp64.json from the `--set full` capture of the five
cfg5 kernels, the ncu summary + launch-list markdown, and copies of the bench / test logs.
Usage: python tools/refresh_records.py <prefix>        (e.g. r2g)"""
import collections
import csv
import io
import json
import os
import re
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pre = sys.argv[1]
G = lambda name: os.path.join(ROOT, "gpurun_out", f"{pre}_{name}")
P = lambda name: os.path.join(ROOT, "profiles", name)
rep = G("cfg5.ncu-rep")

raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
names = ["A_fwd_x", "B_fwd_y", "C_fwd_z_mul_inv_z", "D_inv_y", "E_inv_x_crop"]
num = lambda r, k: float(r[ix[k]].replace(",", ""))
bscale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}[units[ix["dram__bytes_read.sum"]]]
tscale = {"ms": 1, "us": 1e-3, "ns": 1e-6, "msecond": 1, "usecond": 1e-3, "nsecond": 1e-6}[units[ix["gpu__time_duration.sum"]]]
traffic, fp = {}, {}
for n, r in zip(names, data):
    traffic[n] = int(round((num(r, "dram__bytes_read.sum") + num(r, "dram__bytes_write.sum")) * bscale, -3))
    ms = num(r, "gpu__time_duration.sum") * tscale
    pct = num(r, "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active")
    fp[n] = {"ncu_ms": round(ms, 3), "fp64_pipe_pct": pct, "fp64_floor_ms": round(ms * pct / 100, 3)}
t = json.load(open(P("traffic.json")))
t["1536x1536x1536"] = traffic
json.dump(t, open(P("traffic.json"), "w"), indent=1)
f = json.load(open(P("r2_apply_fp64.json")))
f["1536x1536x1536"] = fp
json.dump(f, open(P("r2_apply_fp64.json"), "w"), indent=1)

bench = json.loads(open(G("bench.json")).read().strip().splitlines()[-1])
lrows = [r for r in csv.reader(open(G("launches.csv"))) if len(r) > 5]
lh = next(r for r in lrows if r[0] == "ID")
ik, iv, iu = lh.index("Kernel Name"), lh.index("Metric Value"), lh.index("Metric Unit")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in lrows:
    if not r[0].isdigit():
        continue
    ms = float(r[iv].replace(",", "")) * {"ns": 1e-6, "us": 1e-3, "ms": 1}.get(r[iu], 1)
    name = re.sub(r"\(.*$", "", re.sub(r"^void (fusg::)?", "", r[ik]))
    agg[name][0] += 1
    agg[name][1] += ms
tot = sum(v[1] for v in agg.values())
table = ["| Kernel | launches | total ms | share |", "|---|---|---|---|"]
for k, (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:8]:
    table.append(f"| `{k}` | {n} | {ms:.2f} | {100 * ms / tot:.1f} % |")
cshare = 100 * sum(v[1] for k, v in agg.items() if k.startswith("conv_r16x3")) / tot
summ = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), rep, "768"], capture_output=True, text=True).stdout
pc = bench["passes_ms"]["C_fwd_z_mul_inv_z"]
md = f"""# r2 final: cfg5 (768^3 grid, 1536^3 embedding) apply kernels at the end of round 2

Command: `ncu --set full --import-source on --clock-control none -k regex:"r16x3|conv_r16x3" -c 5 python tools/profile_apply.py 768 1` on one B200 (report gpurun_out/{pre}_cfg5.ncu-rep, not tracked); table by `python tools/ncu_summary.py`. Per launch; `alg` = SURVEY.md 8(d) algorithmic bytes; HBM frac = alg / time / peak (MEASURED_PEAKS.json). ncu serialises launches with cold caches and unthrottled clocks (~1.95 GHz), so its times are below the power-capped bench loop (`profiles/r2_bench.json`: {bench['ms_per_step']:.2f} ms per apply, pass C {pc:.1f} ms, SM clock median {bench['clocks']['sm_mhz']:.0f} MHz, `{', '.join(bench['clocks']['reasons']) or 'no throttle reason'}`).

{summ.strip()}

Kernels: passes A/B `r16x3_row_to_col<4, TMA, 3, FULL>` (box stores, input rows two tiles ahead), pass C `conv_r16x3<1, FULL>` (3 warps per line, quad line order, K^ multiply fused into the last radix 2 in tan form, exchange buffers as 16 rows of 33 entries, radix-16 inner twiddles folded into the butterflies, compiled for full 768-entry rows, 64 CTAs per resident slot), passes D/E `r16x3_col_to_row<4, TMA, 3, FULL>` (box loads, padded exchange rows).

Against `r2_cfg5_tma_ncu_summary.md` (same command before the last session's changes): pass C 26.61 ms at 51.5 % of the FP64 pipe, D/E 7.81 / 3.94 ms, A/B 3.94 / 7.81 ms.

## Launch list of the bench command

`ncu --metrics gpu__time_duration.sum --clock-control none -c 400 python bench.py --headline-only --steps 2 --warmup 1 --no-cpu-baseline --no-cascade` (`r2_final_launches_cfg5.csv`; the host-vector applies run passes A/B/D/E per z-chunk, pass C once):

""" + "\n".join(table) + f"""

Pass C's share of kernel time here ({cshare:.1f} %) agrees with its share of the bench step ({pc:.1f} of {bench['ms_per_step']:.2f} ms, {100 * pc / bench['ms_per_step']:.1f} %).
"""
open(P("r2_final_cfg5_ncu_summary.md"), "w").write(md)
for src, dst in (("launches.csv", "r2_final_launches_cfg5.csv"), ("bench.json", "r2_bench.json"), ("bench_ref.json", "r2_bench_reference.json"),
                 ("pytest.log", "r2_pytest_gpu.log"), ("smoke.log", "r2_smoke.log"), ("configs.json", "r2_configs.json")):
    shutil.copy(G(src), P(dst))
print(json.dumps({"ms_per_step": bench["ms_per_step"], "value": bench["value"], "passes_ms": bench["passes_ms"],
                  "roofline_frac": bench["roofline"]["frac"], "apply_frac": bench["apply_roofline"]["frac"],
                  "e2e": bench["e2e"]["value"], "ncu": fp}, indent=1))
