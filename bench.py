#!/usr/bin/env python
"""Benchmark: volume-potential apply throughput (grid points/s, complex128) on B200.

Workload (BASELINE.json configs[1], "cfg2"): one GreenKernel::apply on a 256^3 grid with a
512^3 circulant embedding, k = 2k_1 at f = 1.1 MHz, c = 1540 m/s, h = lambda_2/6; the source
is a seeded iid complex U[-1,1] field (libstdc++ mt19937, tests/acceptance.cpp:30-36) times a
Gaussian envelope of std 0.2 x box width centred in the box.  A "step" is one apply with the
kernel spectrum cached (include/fus/potential.hpp:25-27); the spectrum build is reported
separately.  Inputs and workspaces (0.27 + 1.6 GB) exceed the 126 MB L2, so no flush is needed.

  python bench.py [--gpus N --steps K --warmup W]       # this framework (libfusg.so)
  python bench.py --impl reference ...                   # the CPU reference path (oracle port)

N > 1 (torchrun): the cfg2 apply is slab-sharded over the ranks (strong scaling): z-slabs of
f/u, x-slabs of the spectrum, two NCCL all-to-all transposes over NVLink per apply
(fusg_kernel_apply_slab); time = max over ranks of CUDA-event time.  --replicas runs
independent per-rank applies instead (weak scaling).
"""
import argparse
import json
import math
import os
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
WORKLOAD = ("cfg2: single volume-potential apply, 256^3 grid, 512^3 circulant embedding, complex128, "
            "k2=2k at f=1.1MHz c=1540, h=lambda2/6, iid U[-1,1] (mt19937 seed 2024) x Gaussian "
            "envelope sigma=0.2*box")
N_SIDE = 256


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def cfg2_inputs():
    from paper_2011_03009_b200 import fus

    c, f0 = 1540.0, 1.1e6
    h = (c / (2 * f0)) / 6.0
    g = fus.make_grid([0, 0, 0], [N_SIDE * h] * 3, h, 2)
    k = fus.Wavenumber(complex(2 * 2 * math.pi * f0 / c, 0.0), 2, 2 * math.pi * f0)
    f = fus.random_vector(g.count(), 2024).reshape(g.dims[2], g.dims[1], g.dims[0])
    cen = 0.5 * (g.lo + g.hi)
    sig = 0.2 * (g.hi[0] - g.lo[0])
    ax = [g.lo[a] + (np.arange(g.dims[a]) + 0.5) * g.dx - cen[a] for a in range(3)]
    r2 = (ax[0] ** 2)[None, None, :] + (ax[1] ** 2)[None, :, None] + (ax[2] ** 2)[:, None, None]
    f = (f * np.exp(-r2 / (2 * sig * sig))).reshape(-1)
    return g, k, f


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


# ------------------------------------------------------------------------- CPU reference arm
def cpu_apply_seconds(g, k, f, workers, max_steps, warmup, budget_s):
    """Oracle port of GreenKernel::apply (src/potential.cpp:120-151) on the host: pocketfft
    on exactly the reference's 2N box. Returns (seconds/apply, steps run)."""
    from oracle import fus_oracle as orc

    orc.build()
    go = orc.VoxelGrid(g.lo, g.hi, g.dx, g.dims, 2)
    K = orc.GreenKernel(go, orc.Wavenumber(k.k, 2, k.omega), workers=workers)
    for _ in range(warmup):
        K.apply(f)
    times = []
    t_all = time.perf_counter()
    while len(times) < max_steps:
        t0 = time.perf_counter()
        K.apply(f)
        times.append(time.perf_counter() - t0)
        if time.perf_counter() - t_all > budget_s:
            break
    return statistics.mean(times), len(times)


def run_reference(args, world, rank):
    if rank != 0:
        return 0
    g, k, f = cfg2_inputs()
    cores = os.cpu_count() or 1
    orc_lib = None
    try:
        from oracle import fus_oracle as orc
        orc_lib = orc.lib()
        orc_lib.orc_set_num_threads(cores)
    except Exception:
        pass
    # every requested warm-up apply runs (~1.4 s each); the timed steps stop after a 150 s budget
    sec, steps = cpu_apply_seconds(g, k, f, cores, args.steps, args.warmup, 150.0)
    v = g.count() / sec
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": steps, "steps_requested": args.steps, "warmup": args.warmup,
        "ms_per_step": sec * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "c128", "data": "synthetic",
        "config": {"workload": WORKLOAD, "grid": [N_SIDE] * 3, "padded": [2 * N_SIDE] * 3,
                   "parallelism": "host cores"},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"{steps} full cfg2 applies (oracle/fus_oracle: pocketfft on the "
                                   f"reference's 2N box, {cores} FFT workers; spectrum prebuilt)"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


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
    return {"config": "cfg4 geometry (bowl R 7.5 cm, l 15 cm, c 1540, rho 1050, beta 4.5, 1 MPa) at "
                      "f0=0.275 MHz, 4096 points, nested n_w=6, 5 harmonics",
            "solve_s": best,
            "grids": [list(cfg.plan.for_harmonic(i).grid.dims) for i in range(2, 6)],
            "rows": [{k: v for k, v in t.__dict__.items()} for t in rows],
            "rayleigh_terms_per_s": n2 * len(cfg.transducer.source_points) / p1 if p1 > 0 else None,
            # FP64 pipe fraction of the Rayleigh sum: 21.25 FP64 instructions per term (SASS of
            # monopole_grid_kernel<0>'s inner loop: 255 per 12 terms) against the pipe's
            # 64 lanes/clk/SM x 148 SMs x 1.965 GHz
            "rayleigh_fp64_pipe_frac": (n2 * len(cfg.transducer.source_points) / p1 * 21.25
                                        / (64 * 148 * 1.965e9)) if p1 > 0 else None}


# ------------------------------------------------------------------------- GPU arm
def run_gpu(args, world, rank, local):
    import torch

    from paper_2011_03009_b200 import _lib, fus

    torch.cuda.set_device(local)
    ctx = fus.context(local)
    g, k, f = cfg2_inputs()
    N = g.count()
    t0 = time.perf_counter()
    K = fus.GreenKernel(g, k, ctx=ctx)
    build_s = time.perf_counter() - t0
    # the same build again: the first one also pays the context's first allocations and module
    # loads; this is the "Evaluate G_k" cost of every further kernel (e.g. each cascade harmonic)
    t0 = time.perf_counter()
    K2 = fus.GreenKernel(g, k, ctx=ctx)
    build_warm_s = time.perf_counter() - t0
    del K2
    P = K.padded
    fd = torch.from_numpy(f).to(f"cuda:{local}")
    ud = torch.empty_like(fd)
    torch.cuda.synchronize()
    L = _lib.lib()
    stream = ctx.stream_ptr

    def step():
        _lib.check(L.fusg_kernel_apply(K.handle, fd.data_ptr(), ud.data_ptr(), 1.0, None))

    for _ in range(max(args.warmup, 3)):
        step()
    ctx.synchronize()

    # ---- timed region: K back-to-back applies on the library stream, CUDA events
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    cs = torch.cuda.ExternalStream(stream)
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
    ms_local = ev0.elapsed_time(ev1) / args.steps
    barrier(world)
    clocks = sampler.stop()
    ms = max_over_ranks(ms_local, world, local)
    value = world * N / (ms * 1e-3)

    # ---- per-pass durations (CUDA events between the passes, same stream)
    pass_ms = (__import__("ctypes").c_double * 5)()
    _lib.check(L.fusg_kernel_apply_timed(K.handle, fd.data_ptr(), ud.data_ptr(), 1.0, 20, pass_ms))
    pass_ms = list(pass_ms)
    per_pass, total_bytes = algorithmic_bytes(g.dims, P)
    names = list(per_pass)
    dom = int(np.argmax(pass_ms))
    hbm, hbm_kind = peaks()
    dom_gbs = per_pass[names[dom]] / (pass_ms[dom] * 1e-3) / 1e9
    traffic = None
    tr_path = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tr_path):
        try:
            traffic = json.load(open(tr_path)).get(names[dom])
        except Exception:
            traffic = None

    # ---- end to end through the C-ABI host-vector call (pinned host buffers, H2D+D2H inside)
    fh = torch.from_numpy(f).pin_memory()
    uh = torch.empty_like(fh).pin_memory()
    for _ in range(2):
        _lib.check(L.fusg_kernel_apply_host(K.handle, fh.data_ptr(), uh.data_ptr(), 1.0))
    e2e_steps = max(3, min(args.steps, 20))
    barrier(world)
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        _lib.check(L.fusg_kernel_apply_host(K.handle, fh.data_ptr(), uh.data_ptr(), 1.0))
    e2e_s = max_over_ranks((time.perf_counter() - t0) / e2e_steps, world, local)

    # parity spot check of the timed output against the host path (same kernels)
    ctx.synchronize()
    assert torch.equal(ud.cpu(), uh), "device and host-vector applies disagree"

    solve = None
    if rank == 0 and not args.no_cascade:
        solve = nested_solve(ctx)
    # evaluate_potential_at at the reference's use (on-axis nodes of a
    # D2-grid field), with the CPU oracle on a bounded sample when the CPU leg runs
    off_grid = vie = acceptance = None
    if rank == 0 and world == 1 and not args.no_cascade:
        from tools import acceptance_bench, potential_at_bench, vie_bench
        off_grid = potential_at_bench.run(cpu_points=0 if args.no_cpu_baseline else 16)
        # a VIE solve at cfg2 size (liver slab), CPU oracle per iteration beside it
        vie = vie_bench.run(cpu=not args.no_cpu_baseline)
        # the reference's long acceptance workloads (recorded wall times in proj/test_output.txt)
        acceptance_bench.criterion1()  # warm-up
        acceptance = {"criterion_1": acceptance_bench.criterion1(), "criterion_6": acceptance_bench.criterion6(),
                      "criterion_10_cascade": acceptance_bench.criterion10_cascade()}

    cpu_baseline = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cores = os.cpu_count() or 1
        try:
            from oracle import fus_oracle as orc
            orc.lib().orc_set_num_threads(cores)
            sec, nst = cpu_apply_seconds(g, k, f, cores, 3, 0, 20.0)
            cpu_baseline = {"value": N / sec, "unit": UNIT, "cores": cores, "kind": "port",
                            "sample": f"{nst} full cfg2 apply(s) by oracle/fus_oracle (pocketfft on the "
                                      f"reference's 2N box, {cores} FFT workers; spectrum prebuilt)"}
        except Exception as e:  # reported, never silently replaced
            cpu_baseline = {"value": None, "unit": UNIT, "cores": cores, "kind": "port",
                            "sample": f"failed: {e}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "c128", "data": "synthetic",
            "config": {"workload": WORKLOAD, "grid": list(g.dims), "padded": list(P),
                       "parallelism": f"replicas{world}" if world > 1 else "single",
                       "l2": "inputs+workspace (1.9 GB) > 126 MB L2; no flush"},
            "roofline": {"bound": "hbm", "kernel": names[dom], "achieved": dom_gbs, "peak": hbm,
                         "peak_kind": hbm_kind, "unit": "GB/s", "frac": dom_gbs / hbm,
                         "traffic": traffic,
                         "algorithmic_bytes_per_launch": per_pass[names[dom]]},
            # pass C is FP64/L1-latency bound, not HBM bound: its FP64 pipe fraction from the
            # SASS instruction count of the 16x16x2 kernel (998 FP64 warp instructions per
            # z-line, ncu: profiles/r1_ncu_summary.md) against 2 per clock per SM
            "pass_c_fp64_pipe": ({"fp64_warp_instr_per_line": 998, "lines": P[0] * P[1],
                                  "frac": 998.0 * P[0] * P[1] / (pass_ms[2] * 1e-3)
                                  / (2 * 148 * 1.965e9)} if tuple(P) == (512, 512, 512) else None),
            "apply_roofline": {"algorithmic_bytes": total_bytes,
                               "achieved_gbs": total_bytes / (ms * 1e-3) / 1e9,
                               "frac": total_bytes / (ms * 1e-3) / 1e9 / hbm},
            "passes_ms": dict(zip(names, pass_ms)),
            "kernel_build_s": build_s, "kernel_build_warm_s": build_warm_s,
            "e2e": {"value": world * N / e2e_s, "unit": UNIT, "h2d_bytes_per_step": 16 * N,
                    "d2h_bytes_per_step": 16 * N},
            "gpu_launches": int(launches),
            "clocks": clocks,
            "cpu_baseline": cpu_baseline,
            "nested_5_harmonic_solve": solve,
            "evaluate_potential_at": off_grid,
            "vie_solve": vie,
            "acceptance": acceptance,
        }
        print(json.dumps(line), flush=True)
    return 0


def run_gpu_sharded(args, world, rank, local):
    """N > 1: one cfg2 apply slab-sharded over all ranks (strong scaling). Rank r owns z-planes
    of f/u and kx columns of the spectrum; the two transposes are NCCL grouped send/recv over
    NVLink (fusg_kernel_apply_slab). Time = max over ranks of CUDA-event time."""
    import ctypes

    import torch
    import torch.distributed as dist

    from paper_2011_03009_b200 import _lib, fus

    torch.cuda.set_device(local)
    ctx = fus.context(local)
    uid = torch.zeros(128, dtype=torch.uint8, device=f"cuda:{local}")
    if rank == 0:
        uid.copy_(torch.frombuffer(bytearray(fus.nccl_unique_id()), dtype=torch.uint8))
    if world > 1:
        dist.broadcast(uid, 0)
    fus.attach_nccl(ctx, world, rank, bytes(uid.cpu().numpy().tobytes()))
    g, k, f = cfg2_inputs()
    N = g.count()
    t0 = time.perf_counter()
    K = fus.SlabKernel(g, k, world, rank, ctx)
    build_s = time.perf_counter() - t0
    # fused peer-store transposes (default when the padded x/y lengths allow): gather every
    # rank's CUDA IPC handles and map the peers' x-slab / A buffers
    transport = args.transport
    if transport == "p2p" and not (set(K_padded(g)[:2]) <= {256, 512, 768, 1024, 1536, 2048}):
        transport = "nccl"
    if transport == "p2p":
        mine = torch.frombuffer(bytearray(K.ipc_handles()), dtype=torch.uint8).to(f"cuda:{local}")
        allh = [torch.empty_like(mine) for _ in range(world)]
        if world > 1:
            dist.all_gather(allh, mine)
        else:
            allh = [mine]
        K.attach_peers(b"".join(bytes(h.cpu().numpy().tobytes()) for h in allh))
    plane = g.dims[0] * g.dims[1]
    f_slab = np.ascontiguousarray(f[K.z0 * plane:(K.z0 + K.nz) * plane])
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
    e2e_steps = max(3, min(args.steps, 20))
    barrier(world)
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        fd.copy_(fh, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        step()
        ctx.synchronize()
        uh.copy_(ud)
    e2e_s = max_over_ranks((time.perf_counter() - t0) / e2e_steps, world, local)
    # all-to-all volume: every rank sends all but its own block in each of the two transposes
    plan = fus.slab_exchange_plan(g, world, rank)
    sent = 2 * 16 * int(plan["a_cnt"].sum() - plan["a_cnt"][rank])
    sent = max_over_ranks(float(sent), world, local)
    per_pass, total_bytes = algorithmic_bytes(g.dims, K_padded(g))
    hbm, hbm_kind = peaks()
    if rank == 0:
        line = {
            "metric": METRIC, "value": N / (ms * 1e-3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "c128",
            "data": "synthetic",
            "transport": transport,
            "config": {"workload": WORKLOAD + ("; z-slab sharded over ranks, transposes fused into passes A/D as "
                                               "NVLink peer stores" if transport == "p2p" else
                                               "; z-slab sharded over ranks, NCCL all-to-all transposes"),
                       "grid": list(g.dims), "padded": list(K_padded(g)),
                       "parallelism": f"slab{world}", "l2": "inputs+workspace > 126 MB L2; no flush"},
            "roofline": {"bound": "hbm+nvlink", "kernel": "sharded apply (passes A-E + 2 transposes)",
                         "achieved": total_bytes / world / (ms * 1e-3) / 1e9, "peak": hbm,
                         "peak_kind": hbm_kind, "unit": "GB/s",
                         "frac": total_bytes / world / (ms * 1e-3) / 1e9 / hbm, "traffic": None,
                         "nvlink_bytes_sent_per_gpu": sent,
                         "nvlink_gbs_if_serialised": sent / (ms * 1e-3) / 1e9,
                         "nvlink_peak_gbs": 770.0},
            "kernel_build_s": build_s,
            "e2e": {"value": N / e2e_s, "unit": UNIT, "h2d_bytes_per_step": 16 * N,
                    "d2h_bytes_per_step": 16 * N},
            "gpu_launches": int(launches), "clocks": clocks, "cpu_baseline": None,
        }
        print(json.dumps(line), flush=True)
    return 0


def K_padded(g):
    from paper_2011_03009_b200 import fus

    return fus.padded_dims(g)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="fusg", choices=["fusg", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-cascade", action="store_true", help="skip the nested 5-harmonic solve")
    ap.add_argument("--sharded", action="store_true", help="use the sharded path even at N = 1")
    ap.add_argument("--transport", default="p2p", choices=["p2p", "nccl"],
                    help="sharded apply: transposes fused into passes A/D as peer stores, or NCCL all-to-all")
    ap.add_argument("--replicas", action="store_true",
                    help="N > 1: independent per-rank applies (weak scaling) instead of the sharded apply")
    args = ap.parse_args()
    world, rank, local = dist_setup(args)
    try:
        if args.impl == "reference":
            return run_reference(args, world, rank)
        if (world > 1 or args.sharded) and not args.replicas:
            return run_gpu_sharded(args, world, rank, local)
        return run_gpu(args, world, rank, local)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
