#!/usr/bin/env python
"""Benchmark: volume-potential apply throughput (grid points/s, complex128) on B200.

Headline workload (BASELINE.json configs[4], "cfg5", the largest configuration that fits one
GPU): one GreenKernel::apply on a 768^3 grid with a 1536^3 circulant embedding (~58 GB in the
reference's form), k h = pi/3 (h = lambda/6 at f = 1.1 MHz, c = 1540 m/s), source = seeded iid
complex U[-1,1] (libstdc++ mt19937 seed 768, tests/acceptance.cpp:30-36).  A "step" is one
apply with the kernel spectrum cached (include/fus/potential.hpp:25-27); the spectrum build is
reported separately.  Inputs (7.25 GB) and workspaces (43.5 GB) exceed the 126 MB L2, so no
flush is needed.  cfg2 (256^3 / 512^3) is measured beside it as an extra key.

  python bench.py [--gpus N --steps K --warmup W]       # this framework (libfusg.so)
  python bench.py --impl reference ...                   # the reference's CPU path (oracle port)

--gpus N > 1 without a torchrun environment re-launches itself under torch.distributed.run
with N ranks.  N > 1: the cfg5 apply is slab-sharded over the ranks (strong scaling): z-slabs
of f/u, x-slabs of the spectrum, the two 3D-FFT transposes fused into passes A/D as NVLink
peer stores (fusg_kernel_apply_slab_p2p); time = max over ranks of CUDA-event time.

The reference arm never imports the framework package (no libfusg.so): its inputs come from
oracle/ and its config dict is the same object as the GPU arm's.
"""
import argparse
import json
import math
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "volume-potential grid pts/s (c128)"
UNIT = "grid_pts/s"

# ---- workloads (plain constants: both arms build their config from these alone)
C0, F0 = 1540.0, 1.1e6
CFG5 = {"n": 768, "harmonic": 1, "seed": 768,
        "workload": ("cfg5: single volume-potential apply, 768^3 grid, 1536^3 circulant embedding, "
                     "complex128, k=2*pi*f/c at f=1.1MHz c=1540 (k h = pi/3, h = lambda/6), "
                     "iid U[-1,1] source (mt19937 seed 768)")}
CFG2 = {"n": 256, "harmonic": 2, "seed": 2024,
        "workload": ("cfg2: single volume-potential apply, 256^3 grid, 512^3 circulant embedding, complex128, "
                     "k2=2k at f=1.1MHz c=1540, h=lambda2/6, iid U[-1,1] (mt19937 seed 2024) x Gaussian "
                     "envelope sigma=0.2*box")}


def geometry(cfg):
    """(h, k, omega) of a cube workload: h = lambda_n / 6, k = n * 2 pi f / c (real)."""
    n = cfg["harmonic"]
    h = (C0 / (n * F0)) / 6.0
    return h, n * 2 * math.pi * F0 / C0, 2 * math.pi * F0


def bench_config(cfg, world):
    n = cfg["n"]
    return {"workload": cfg["workload"], "grid": [n] * 3, "padded": [2 * n] * 3, "seed": cfg["seed"],
            "parallelism": "single" if world == 1 else f"zslab{world}",
            "l2": "inputs+workspace > 126 MB L2; no flush"}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 7672.0, "fallback (B200_PROFILING.md)"


def gpu_inputs(cfg):
    from paper_2011_03009_b200 import fus

    h, k, om = geometry(cfg)
    n = cfg["n"]
    g = fus.make_grid([0, 0, 0], [n * h] * 3, h, cfg["harmonic"])
    kw = fus.Wavenumber(complex(k, 0.0), cfg["harmonic"], om)
    f = fus.random_vector(g.count(), cfg["seed"])
    if cfg is CFG2:
        f = envelope(f, g.lo, g.hi, g.dx, g.dims)
    return g, kw, f


def envelope(f, lo, hi, dx, dims):
    f = f.reshape(dims[2], dims[1], dims[0])
    cen = 0.5 * (np.asarray(lo) + np.asarray(hi))
    sig = 0.2 * (hi[0] - lo[0])
    ax = [lo[a] + (np.arange(dims[a]) + 0.5) * dx - cen[a] for a in range(3)]
    r2 = (ax[0] ** 2)[None, None, :] + (ax[1] ** 2)[None, :, None] + (ax[2] ** 2)[:, None, None]
    return (f * np.exp(-r2 / (2 * sig * sig))).reshape(-1)


def algorithmic_bytes(N, P):
    """pruned fused 5-pass pipeline, 16 B per complex128 element."""
    Nx, Ny, Nz = N
    Px, Py, Pz = P
    n = Nx * Ny * Nz
    k_oct = (Px // 2 + 1) * (Py // 2 + 1) * (Pz // 2 + 1)
    per_pass = {
        "A_fwd_x": 16 * (n + Px * Ny * Nz),
        "B_fwd_y": 16 * (Px * Ny * Nz + Px * Py * Nz),
        "C_fwd_z_mul_inv_z": 16 * (2 * Px * Py * Nz + k_oct),
        "D_inv_y": 16 * (Px * Py * Nz + Px * Ny * Nz),
        "E_inv_x_crop": 16 * (Px * Ny * Nz + n),
    }
    return per_pass, sum(per_pass.values())


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ["clocks.sm", "clocks.max.sm", "power.draw", "clocks_event_reasons.active",
              "clocks_event_reasons.hw_slowdown", "clocks_event_reasons.hw_thermal_slowdown",
              "clocks_event_reasons.sw_thermal_slowdown", "clocks_event_reasons.sw_power_cap"]

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist

        backend = "nccl" if torch.cuda.is_available() else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(local)
        dist.init_process_group(backend)
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def max_over_ranks(x, world, local):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    dev = f"cuda:{local}" if torch.cuda.is_available() else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def relaunch_under_torchrun(n):
    """--gpus N > 1 outside torchrun: run this script again as N ranks (one per GPU)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


# ------------------------------------------------------------------------- CPU reference arm
SAMPLE_PLANES = 32


def cpu_sampled(cfg, workers, steps, warmup, budget_s):
    """The reference's apply (src/potential.cpp:120-151) by the oracle port on the host, as a
    bounded sample: SAMPLE_PLANES z-planes' share of every stage of the P-box apply at the full
    line lengths (oracle.SampledApply), extrapolated to the whole apply.  Returns
    (mean seconds per extrapolated apply, steps run, fraction, mean seconds per sample)."""
    from oracle import fus_oracle as orc

    orc.build()
    n = cfg["n"]
    s = orc.SampledApply([n] * 3, [2 * n] * 3, SAMPLE_PLANES, workers, cfg["seed"])
    for _ in range(warmup):
        s.run()
    t_all, raw = time.perf_counter(), []
    while len(raw) < max(1, steps):
        raw.append(s.run())
        if time.perf_counter() - t_all > budget_s:
            break
    mean = statistics.mean(raw)
    return mean / s.fraction, len(raw), s.fraction, mean


def cpu_baseline_record(cfg, steps, warmup, budget_s, one_thread=True):
    cores = os.cpu_count() or 1
    from oracle import fus_oracle as orc

    orc.lib().orc_set_num_threads(cores)
    sec, nst, frac, raw = cpu_sampled(cfg, cores, steps, warmup, budget_s)
    n = cfg["n"] ** 3
    rec = {"value": n / sec, "unit": UNIT, "cores": cores, "kind": "port",
           "sample": (f"{nst} sample(s) of the reference apply (oracle port: pad, pocketfft x/y/z line batches "
                      f"fwd+inv, spectrum multiply, 1/|P| scale, crop) on {SAMPLE_PLANES} of {2 * cfg['n']} "
                      f"z-planes' share of every stage (fraction {frac:.5f}), {cores} FFT workers, "
                      f"{raw:.3f} s per sample; extrapolated = sample / fraction"),
           "extrapolated": True, "seconds_per_apply": sec, "steps_run": nst}
    if one_thread:
        # the reference's own FFT is single-threaded FFTW (proj/CMakeLists.txt:11,29): the
        # faithful mirror, reported beside the all-core variant
        s1, _, _, raw1 = cpu_sampled(cfg, 1, 1, 0, 1e9)
        rec["fft_1thread"] = {"value": n / s1, "unit": UNIT, "cores": 1, "seconds_per_apply": s1,
                              "sample": f"1 sample, 1 FFT worker, {raw1:.3f} s per sample, extrapolated"}
    return rec


def host_info():
    info = {"nproc": os.cpu_count()}
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                info["cpu"] = ln.split(":", 1)[1].strip()
                break
        for ln in open("/proc/meminfo"):
            if ln.startswith("MemTotal"):
                info["mem_total"] = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return info


def run_reference(args, world, rank):
    if rank != 0:
        return 0
    cfg = CFG5
    rec = cpu_baseline_record(cfg, args.steps, args.warmup, 240.0, one_thread=True)
    n = cfg["n"] ** 3
    sec = rec["seconds_per_apply"]
    line = {
        "impl": "reference", "metric": METRIC, "value": rec["value"], "unit": UNIT, "n_gpus": world,
        "steps": rec["steps_run"], "steps_requested": args.steps, "warmup": args.warmup,
        "ms_per_step": sec * 1e3, "higher_is_better": True, "scaling": "weak" if world == 1 else "strong",
        "vs_baseline": None, "dtype": "c128", "data": "synthetic",
        "config": bench_config(cfg, world),
        "cpu_baseline": rec,
        "host": host_info(),
        "e2e": {"value": rec["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": "host-vector apply by definition (the reference is CPU-only); n=%d voxels" % n,
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------- GPU helpers
def nested_solve(ctx, reps=2):
    """BASELINE metric part 2: wall time of the nested 5-harmonic recursion (run_cascade) on
    config 4's geometry at the desk frequency 0.275 MHz (full size needs >= 4 GPUs: SURVEY.md
    8(e)). Best of `reps` after one warm-up; per-stage rows come from CUDA events."""
    import torch

    from paper_2011_03009_b200 import fus
    from tools import cascades

    cfg = cascades.cfg4(fus, desk=True)
    fus.run_cascade(cfg, ctx=ctx)
    best, rows = None, None
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = fus.run_cascade(cfg, ctx=ctx)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if best is None or dt < best:
            best, rows = dt, r.timings
    n2 = cfg.plan.for_harmonic(2).grid.count()
    p1 = rows[0].p1_s
    fp64 = rayleigh_fp64_profile()
    tps = n2 * len(cfg.transducer.source_points) / p1 if p1 > 0 else None
    return {"config": "cfg4 geometry (bowl R 7.5 cm, l 15 cm, c 1540, rho 1050, beta 4.5, 1 MPa) at "
                      "f0=0.275 MHz, 4096 points, nested n_w=6, 5 harmonics",
            "solve_s": best,
            "grids": [list(cfg.plan.for_harmonic(i).grid.dims) for i in range(2, 6)],
            "rows": [{k: v for k, v in t.__dict__.items()} for t in rows],
            "rayleigh_terms_per_s": tps,
            # FP64 pipe fraction of the Rayleigh sum: ncu-measured FP64 warp instructions per
            # term (profiles/, same kernel build) x terms/s against 2 warp instructions per clock
            # per SM x 148 SMs x the SM clock
            "rayleigh_fp64_pipe_frac": (tps * fp64["fp64_thread_instr_per_term"] / (64 * 148 * 1.965e9))
                                       if (tps and fp64) else None,
            "rayleigh_fp64_source": fp64}


def rayleigh_fp64_profile():
    p = os.path.join(ROOT, "profiles", "r2_rayleigh_fp64.json")
    try:
        return json.load(open(p))
    except Exception:
        return None


def measure_apply(cfg, ctx, steps, warmup, world, local, sampler_on=True, e2e_steps=3):
    """Device-resident apply on one GPU: K timed steps (CUDA events on the library stream),
    per-pass events, e2e through the public host-vector call (pageable numpy, the
    GreenKernel::apply(VectorXcd) drop-in) and pinned."""
    import ctypes

    import torch

    from paper_2011_03009_b200 import _lib, fus

    g, k, f = gpu_inputs(cfg)
    N = g.count()
    t0 = time.perf_counter()
    K = fus.GreenKernel(g, k, ctx=ctx)
    ctx.synchronize()
    build_s = time.perf_counter() - t0
    P = K.padded
    dev = f"cuda:{local}"
    fd = torch.from_numpy(f).to(dev)
    ud = torch.empty_like(fd)
    torch.cuda.synchronize()
    L = _lib.lib()

    def step():
        _lib.check(L.fusg_kernel_apply(K.handle, fd.data_ptr(), ud.data_ptr(), 1.0, None))

    for _ in range(max(warmup, 3)):
        step()
    ctx.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    cs = torch.cuda.ExternalStream(ctx.stream_ptr)
    sampler = ClockSampler(local) if sampler_on else None
    if sampler:
        sampler.start()
        time.sleep(0.3)
    barrier(world)
    ctx.synchronize()
    launches0 = ctx.launch_count()
    ev0.record(cs)
    for _ in range(steps):
        step()
    ev1.record(cs)
    ev1.synchronize()
    launches = ctx.launch_count() - launches0
    ms = ev0.elapsed_time(ev1) / steps
    barrier(world)
    clocks = sampler.stop() if sampler else None

    pass_ms = (ctypes.c_double * 5)()
    _lib.check(L.fusg_kernel_apply_timed(K.handle, fd.data_ptr(), ud.data_ptr(), 1.0, 3, pass_ms))
    pass_ms = list(pass_ms)

    # end to end through the public host-vector API (f and u in pageable host memory, the
    # reference's VectorXcd case; H2D + apply + D2H inside the timed region, chunk-pipelined
    # through the library's pinned staging ring), then the same with pinned host buffers
    u_host = np.empty_like(f)
    K.apply_host(f, out=u_host)
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        K.apply_host(f, out=u_host)
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    fh = torch.from_numpy(f).pin_memory()
    uh = torch.empty_like(fh).pin_memory()
    _lib.check(L.fusg_kernel_apply_host(K.handle, fh.data_ptr(), uh.data_ptr(), 1.0))
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        _lib.check(L.fusg_kernel_apply_host(K.handle, fh.data_ptr(), uh.data_ptr(), 1.0))
    e2e_pinned_s = (time.perf_counter() - t0) / e2e_steps
    ctx.synchronize()
    # the timed device output, the pageable and the pinned host paths run the same kernels
    same = bool(torch.equal(ud.cpu(), uh)) and bool(np.array_equal(u_host, uh.numpy()))
    del fh, uh, u_host
    out = {"N": N, "dims": list(g.dims), "P": list(P), "ms": ms, "pass_ms": pass_ms, "launches": launches,
           "clocks": clocks, "build_s": build_s, "e2e_s": e2e_s, "e2e_pinned_s": e2e_pinned_s,
           "paths_bitwise_equal": same}
    del K, fd, ud
    torch.cuda.empty_cache()
    return out


def roofline_of(m):
    per_pass, total = algorithmic_bytes(m["dims"], m["P"])
    names = list(per_pass)
    dom = int(np.argmax(m["pass_ms"]))
    hbm, kind = peaks()
    gbs = per_pass[names[dom]] / (m["pass_ms"][dom] * 1e-3) / 1e9
    traffic = None
    try:
        tr = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
        key = "x".join(str(p) for p in m["P"])
        traffic = tr.get(key, {}).get(names[dom]) if key in tr else None
    except Exception:
        pass
    roof = {"bound": "hbm", "kernel": names[dom], "achieved": gbs, "peak": hbm, "peak_kind": kind,
            "unit": "GB/s", "frac": gbs / hbm, "traffic": traffic,
            "algorithmic_bytes_per_launch": per_pass[names[dom]],
            "launch_ms": m["pass_ms"][dom], "share_of_step": m["pass_ms"][dom] / sum(m["pass_ms"])}
    # the dominant kernel against its binding floor, max(HBM floor, FP64 floor): the FP64 floor is
    # the ncu-measured FP64-pipe time of the same kernel at 100 % (profiles/r2_apply_fp64.json)
    try:
        fp = json.load(open(os.path.join(ROOT, "profiles", "r2_apply_fp64.json")))
        key = "x".join(str(p) for p in m["P"])
        if key in fp and names[dom] in fp[key]:
            hbm_floor = per_pass[names[dom]] / (hbm * 1e9) * 1e3
            fp64_floor = fp[key][names[dom]]["fp64_floor_ms"]
            roof["binding_floor"] = {"hbm_ms": hbm_floor, "fp64_ms": fp64_floor,
                                     "bound": "fp64" if fp64_floor > hbm_floor else "hbm",
                                     "frac": max(hbm_floor, fp64_floor) / m["pass_ms"][dom],
                                     "source": "profiles/r2_apply_fp64.json"}
    except Exception:
        pass
    apply_roof = {"algorithmic_bytes": total, "achieved_gbs": total / (m["ms"] * 1e-3) / 1e9,
                  "frac": total / (m["ms"] * 1e-3) / 1e9 / hbm,
                  "per_pass_frac": {nm: per_pass[nm] / (t * 1e-3) / 1e9 / hbm
                                    for nm, t in zip(names, m["pass_ms"])}}
    return roof, apply_roof, dict(zip(names, m["pass_ms"]))


# ------------------------------------------------------------------------- GPU arm (N = 1)
def run_gpu(args, world, rank, local):
    import torch

    from paper_2011_03009_b200 import fus

    torch.cuda.set_device(local)
    ctx = fus.context(local)
    m = measure_apply(CFG5, ctx, args.steps, args.warmup, world, local)
    N = m["N"]
    value = world * N / (m["ms"] * 1e-3)
    roof, apply_roof, passes = roofline_of(m)

    extras = {}
    if not args.headline_only:
        m2 = measure_apply(CFG2, ctx, 50, 3, world, local, sampler_on=False)
        r2, a2, p2 = roofline_of(m2)
        extras["cfg2"] = {"workload": CFG2["workload"], "value": m2["N"] / (m2["ms"] * 1e-3), "unit": UNIT,
                          "ms_per_step": m2["ms"], "steps": 50, "roofline": r2, "apply_roofline": a2,
                          "passes_ms": p2, "e2e_pageable": m2["N"] / m2["e2e_s"],
                          "e2e_pinned": m2["N"] / m2["e2e_pinned_s"], "kernel_build_s": m2["build_s"]}
    if rank == 0 and not args.no_cascade:
        extras["nested_5_harmonic_solve"] = nested_solve(ctx)
    if rank == 0 and world == 1 and not args.no_cascade and not args.headline_only:
        from tools import acceptance_bench, potential_at_bench, vie_bench
        # evaluate_potential_at at the reference's use
        extras["evaluate_potential_at"] = potential_at_bench.run(cpu_points=0 if args.no_cpu_baseline else 16)
        # a VIE solve at cfg2 size (liver slab)
        extras["vie_solve"] = vie_bench.run(cpu=not args.no_cpu_baseline)
        acceptance_bench.criterion1()  # warm-up
        extras["acceptance"] = {"criterion_1": acceptance_bench.criterion1(),
                                "criterion_6": acceptance_bench.criterion6(),
                                "criterion_10_cascade": acceptance_bench.criterion10_cascade()}

    cpu_baseline = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu_baseline = cpu_baseline_record(CFG5, 3, 1, 20.0, one_thread=True)
        except Exception as e:  # reported, never silently replaced
            cpu_baseline = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
                            "sample": f"failed: {e}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": m["ms"], "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "c128", "data": "synthetic",
            "config": bench_config(CFG5, world),
            "roofline": roof,
            "apply_roofline": apply_roof,
            "passes_ms": passes,
            "kernel_build_s": m["build_s"],
            "e2e": {"value": world * N / m["e2e_s"], "unit": UNIT, "h2d_bytes_per_step": 16 * N,
                    "d2h_bytes_per_step": 16 * N,
                    "path": "GreenKernel.apply_host on pageable numpy buffers (fusg_kernel_apply_host)",
                    "pinned_value": world * N / m["e2e_pinned_s"]},
            "gpu_launches": int(m["launches"]),
            "clocks": m["clocks"],
            "cpu_baseline": cpu_baseline,
            "host": host_info(),
            "paths_bitwise_equal": m["paths_bitwise_equal"],
        }
        line.update(extras)
        print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------- GPU arm (N > 1)
def run_gpu_sharded(args, world, rank, local):
    """N > 1: one cfg5 apply slab-sharded over all ranks (strong scaling). Rank r owns z-planes
    of f/u and kx columns of the spectrum; the two transposes are fused into passes A/D as NVLink
    peer stores (or NCCL grouped send/recv with --transport nccl). Time = max over ranks of
    CUDA-event time."""
    import torch
    import torch.distributed as dist

    from paper_2011_03009_b200 import _lib, fus

    cfg = CFG5 if not args.cfg2 else CFG2
    torch.cuda.set_device(local)
    ctx = fus.context(local)
    uid = torch.zeros(128, dtype=torch.uint8, device=f"cuda:{local}")
    if rank == 0:
        uid.copy_(torch.frombuffer(bytearray(fus.nccl_unique_id()), dtype=torch.uint8))
    if world > 1:
        dist.broadcast(uid, 0)
    fus.attach_nccl(ctx, world, rank, bytes(uid.cpu().numpy().tobytes()))
    h, kk, om = geometry(cfg)
    n = cfg["n"]
    g = fus.make_grid([0, 0, 0], [n * h] * 3, h, cfg["harmonic"])
    k = fus.Wavenumber(complex(kk, 0.0), cfg["harmonic"], om)
    N = g.count()
    t0 = time.perf_counter()
    K = fus.SlabKernel(g, k, world, rank, ctx)
    build_s = time.perf_counter() - t0
    transport = args.transport
    P = fus.padded_dims(g)
    if transport == "p2p" and not (set(P[:2]) <= {256, 512, 768, 1024, 1536, 2048}):
        transport = "nccl"
    if transport == "p2p":
        mine = torch.frombuffer(bytearray(K.ipc_handles()), dtype=torch.uint8).to(f"cuda:{local}")
        allh = [torch.empty_like(mine) for _ in range(world)]
        if world > 1:
            dist.all_gather(allh, mine)
        else:
            allh = [mine]
        K.attach_peers(b"".join(bytes(x.cpu().numpy().tobytes()) for x in allh))
    plane = g.dims[0] * g.dims[1]
    # this rank's z-slab of the seeded source (the mt19937 stream is sequential in x-fastest order)
    f_pre = fus.random_vector((K.z0 + K.nz) * plane, cfg["seed"])
    f_slab = np.ascontiguousarray(f_pre[K.z0 * plane:])
    del f_pre
    fd = torch.from_numpy(f_slab).to(f"cuda:{local}")
    ud = torch.empty_like(fd)
    L = _lib.lib()
    apply_fn = L.fusg_kernel_apply_slab_p2p if transport == "p2p" else L.fusg_kernel_apply_slab

    def step():
        _lib.check(apply_fn(K.handle, fd.data_ptr(), ud.data_ptr(), 1.0, None))

    for _ in range(max(args.warmup, 3)):
        step()
    ctx.synchronize()
    cs = torch.cuda.ExternalStream(ctx.stream_ptr)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    barrier(world)
    ctx.synchronize()
    launches0 = ctx.launch_count()
    ev0.record(cs)
    for _ in range(args.steps):
        step()
    ev1.record(cs)
    ev1.synchronize()
    launches = ctx.launch_count() - launches0
    ms = max_over_ranks(ev0.elapsed_time(ev1) / args.steps, world, local)
    barrier(world)
    clocks = sampler.stop()
    # end to end through the public API: pinned host slab -> device, sharded apply, -> host
    fh = torch.from_numpy(f_slab).pin_memory()
    uh = torch.empty_like(fh).pin_memory()
    e2e_steps = 3
    barrier(world)
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        fd.copy_(fh, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        step()
        ctx.synchronize()
        uh.copy_(ud)
    e2e_s = max_over_ranks((time.perf_counter() - t0) / e2e_steps, world, local)
    plan = fus.slab_exchange_plan(g, world, rank)
    sent = 2 * 16 * int(plan["a_cnt"].sum() - plan["a_cnt"][rank])
    sent = max_over_ranks(float(sent), world, local)
    per_pass, total_bytes = algorithmic_bytes(g.dims, P)
    hbm, hbm_kind = peaks()
    nvl = 770.0  # measured peer copy per direction (B200_PROFILING.md); 900 GB/s nominal
    del K, fd, ud, fh, uh
    torch.cuda.empty_cache()
    # the nested 5-harmonic recursion sharded over the ranks (paper_2011_03009_b200/zslab.py):
    # config 4's geometry at the desk frequency by default, the full 1.1 MHz config with
    # --cascade-full (per-GPU memory budget)
    solve = None
    if not args.no_cascade:
        from paper_2011_03009_b200 import zslab
        from tools import cascades

        ccfg = cascades.cfg4(fus, desk=not args.cascade_full)
        comm = zslab.Comm()
        if not args.cascade_full:
            zslab.run_cascade_zslab(ccfg, comm, ctx)  # warm-up
        rc = zslab.run_cascade_zslab(ccfg, comm, ctx)
        solve = {"config": ("cfg4 geometry (bowl R 7.5 cm, l 15 cm, c 1540, rho 1050, beta 4.5, 1 MPa), "
                            f"f0={ccfg.transducer.f0 / 1e6:g} MHz, 4096 points, nested n_w=6, 5 harmonics"),
                 "solve_s": rc.solve_s, "grids": [list(gr.dims) for gr in rc.grids], "rows": rc.rows,
                 "sharding": f"zslab{world}", "time": "wall clock of the whole recursion, max over ranks"}
        del rc
        torch.cuda.empty_cache()
    if rank == 0:
        line = {
            "metric": METRIC, "value": N / (ms * 1e-3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "c128",
            "data": "synthetic", "transport": transport,
            "config": bench_config(cfg, world),
            "roofline": {"bound": "hbm+nvlink", "kernel": "sharded apply (passes A-E + 2 transposes)",
                         "achieved": total_bytes / world / (ms * 1e-3) / 1e9, "peak": hbm,
                         "peak_kind": hbm_kind, "unit": "GB/s",
                         "frac": total_bytes / world / (ms * 1e-3) / 1e9 / hbm, "traffic": None,
                         "nvlink_bytes_sent_per_gpu": sent,
                         "nvlink_gbs_if_serialised": sent / (ms * 1e-3) / 1e9,
                         "nvlink_peak_gbs": nvl, "nvlink_peak_kind": "measured peer copy (900 nominal)",
                         "nvlink_frac_if_serialised": sent / (ms * 1e-3) / 1e9 / nvl},
            "kernel_build_s": build_s,
            "e2e": {"value": N / e2e_s, "unit": UNIT, "h2d_bytes_per_step": 16 * N,
                    "d2h_bytes_per_step": 16 * N},
            "gpu_launches": int(launches), "clocks": clocks, "cpu_baseline": None,
            "nested_5_harmonic_solve": solve,
        }
        print(json.dumps(line), flush=True)
    return 0


def main():
    # NCCL prints its version banner on stdout at communicator creation when NCCL_DEBUG asks for
    # it; the contract is one JSON line on rank 0's stdout, so keep NCCL's chatter at warnings
    if not os.environ.get("FUSG_KEEP_NCCL_DEBUG") and os.environ.get("NCCL_DEBUG", "").upper() in ("", "VERSION", "INFO", "TRACE"):
        os.environ["NCCL_DEBUG"] = "WARN"
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="fusg", choices=["fusg", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-cascade", action="store_true", help="skip the nested 5-harmonic solve")
    ap.add_argument("--headline-only", action="store_true", help="cfg5 line only (no cfg2 / 8(f) extras)")
    ap.add_argument("--sharded", action="store_true", help="use the sharded path even at N = 1")
    ap.add_argument("--cfg2", action="store_true", help="sharded path on cfg2 instead of cfg5")
    ap.add_argument("--cascade-full", action="store_true",
                    help="N > 1: the sharded nested solve on the full 1.1 MHz config 4 (needs >= 4 GPUs)")
    ap.add_argument("--transport", default="p2p", choices=["p2p", "nccl"],
                    help="sharded apply: transposes fused into passes A/D as peer stores, or NCCL all-to-all")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch_under_torchrun(args.gpus)
    world, rank, local = dist_setup(args)
    try:
        if args.impl == "reference":
            return run_reference(args, world, rank)
        if world > 1 or args.sharded:
            return run_gpu_sharded(args, world, rank, local)
        return run_gpu(args, world, rank, local)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
