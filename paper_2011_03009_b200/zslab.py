"""Multi-process z-slab sharded harmonic recursion: run_cascade
(src/cascade.cpp:42-107) with one process per GPU, every field split into z-slabs.

Per harmonic i, rank r owns planes [z0_r, z0_r + nz_r) of grid i (ragged: the first
Nz mod G ranks take one more plane, the same split as the slab-sharded apply):

* p1: the incident field of its own slab (fusg_monopole_grid_zslab), no collective; the power
  normalisation is evaluated by every rank (deterministic, fixed-order reduction).
* transfers between nested grids: the target slab reads one contiguous source plane range
  (fusg_interpolate_source_planes, a host restatement of the device's z cell, src/grid.cpp:
  156-170); the planes a rank does not own arrive from their owners by point-to-point
  send / recv (NCCL on GPUs, gloo on CPU), then fusg_interpolate_zslab transfers the slab;
* rhs_source: elementwise on the slab;
* the apply: the slab-sharded operator (SlabKernel), transposes as NCCL all-to-alls or fused
  into passes A / D as NVLink peer stores.

Every stage uses the same kernels as the single-GPU path, so the gathered fields equal
run_cascade's bit for bit (tested with one NCCL rank on the B200, and in loopback).
"""
from __future__ import annotations

import time
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Tuple

from . import fus

try:
    import torch
    import torch.distributed as dist
except ImportError:  # pragma: no cover - torch is part of the image
    torch = None
    dist = None


def zsplit(n: int, G: int) -> List[Tuple[int, int]]:
    """[(z0, nz)] of n planes over G ranks (the first n mod G ranks take one more)."""
    return fus._zsplit(n, G)


def transfer_plan(src: "fus.VoxelGrid", tgt: "fus.VoxelGrid", G: int):
    """Halo plan of one nested-grid transfer.  need[r] = (lo, hi): the source planes target
    slab r reads (None for an empty slab); parts[(q, r)] = (a, b): the planes [a, b) of source
    slab q that rank r needs (q == r included)."""
    s_sl, t_sl = zsplit(src.dims[2], G), zsplit(tgt.dims[2], G)
    need: List[Optional[Tuple[int, int]]] = []
    for z0, nz in t_sl:
        need.append(fus.interpolate_source_planes(src, tgt, z0, nz) if nz > 0 else None)
    parts: Dict[Tuple[int, int], Tuple[int, int]] = {}
    for r, nr in enumerate(need):
        if nr is None:
            continue
        lo, hi = nr
        for q, (qz0, qnz) in enumerate(s_sl):
            a, b = max(lo, qz0), min(hi + 1, qz0 + qnz)
            if a < b:
                parts[(q, r)] = (a, b)
    return need, parts


class Comm:
    """The point-to-point exchange of the transfers over a torch.distributed process group
    (NCCL for CUDA tensors, gloo for CPU tensors)."""

    def __init__(self, group=None):
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1

    def exchange(self, sends: Dict[int, "torch.Tensor"], recvs: Dict[int, "torch.Tensor"]):
        """Send sends[peer] to peer and receive recvs[peer] (preallocated) from peer, batched."""
        ops = []
        for peer, t in sends.items():
            ops.append(dist.P2POp(dist.isend, _wire(t), peer, self.group))
        for peer, t in recvs.items():
            ops.append(dist.P2POp(dist.irecv, _wire(t), peer, self.group))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()

    def max(self, x: float) -> float:
        if self.world == 1:
            return x
        dev = "cuda" if (torch.cuda.is_available() and dist.get_backend(self.group) == "nccl") else "cpu"
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        return float(t.item())

    def all_gather_bytes(self, b: bytes) -> bytes:
        if self.world == 1:
            return b
        dev = "cuda" if dist.get_backend(self.group) == "nccl" else "cpu"
        mine = torch.frombuffer(bytearray(b), dtype=torch.uint8).to(dev)
        allb = [torch.empty_like(mine) for _ in range(self.world)]
        dist.all_gather(allb, mine, group=self.group)
        return b"".join(bytes(x.cpu().numpy().tobytes()) for x in allb)

    def barrier(self):
        if self.world > 1:
            dist.barrier(group=self.group)


def _wire(t):
    """complex128 tensors travel as float64 pairs (gloo has no complex type)."""
    return torch.view_as_real(t) if t.is_complex() else t


def gather_source_planes(comm: Comm, src: "fus.VoxelGrid", tgt: "fus.VoxelGrid", my_slab, plan=None):
    """This rank's contiguous source plane range (lo, planes tensor) for its target slab: its own
    planes plus the halo planes received from their owners; every rank sends what the others
    need.  my_slab holds this rank's planes of the source field (x fastest)."""
    G, r = comm.world, comm.rank
    need, parts = plan or transfer_plan(src, tgt, G)
    s_z0 = zsplit(src.dims[2], G)[r][0]
    pl = int(src.dims[0]) * int(src.dims[1])
    sends = {dst: my_slab[(a - s_z0) * pl:(b - s_z0) * pl].contiguous()
             for (q, dst), (a, b) in parts.items() if q == r and dst != r}
    if need[r] is None:
        comm.exchange(sends, {})
        return None, None
    lo, hi = need[r]
    out = torch.empty((hi + 1 - lo) * pl, dtype=my_slab.dtype, device=my_slab.device)
    recvs = {}
    for (q, dst), (a, b) in parts.items():
        if dst != r:
            continue
        view = out[(a - lo) * pl:(b - lo) * pl]
        if q == r:
            view.copy_(my_slab[(a - s_z0) * pl:(b - s_z0) * pl])
        else:
            recvs[q] = view
    comm.exchange(sends, recvs)
    return lo, out


@dataclass
class SlabCascade:
    """This rank's share of a sharded run_cascade: slabs[n - 1] holds planes slabs_z[n - 1] of
    harmonic n on grids[n - 1]; rows carry the stage times (max over ranks)."""
    grids: List["fus.VoxelGrid"] = field(default_factory=list)
    slabs: List["torch.Tensor"] = field(default_factory=list)
    slabs_z: List[Tuple[int, int]] = field(default_factory=list)
    source_normalization: float = 1.0
    rows: List[dict] = field(default_factory=list)
    solve_s: float = 0.0


def run_cascade_zslab(cfg: "fus.CascadeConfig", comm: Comm, ctx: Optional["fus.Context"] = None,
                      transport: str = "auto") -> SlabCascade:
    """run_cascade (src/cascade.cpp:42-107) on this rank's z-slabs; every rank of comm calls it.
    The context must have an NCCL communicator attached (fus.attach_nccl) when comm.world > 1
    or transport is not "loopback"."""
    ctx = ctx or fus.context()
    n = int(cfg.n_harmonics)
    if n < 2:
        raise ValueError("run_cascade: n_harmonics must be >= 2")
    G, r = comm.world, comm.rank
    t, med = cfg.transducer, cfg.medium
    grid_of = lambda i: cfg.plan.for_harmonic(max(i, 2)).grid  # p1 lives on D_2's grid
    for i in range(2, n + 1):
        if grid_of(i).dims[2] < G:
            raise ValueError("run_cascade_zslab: every grid needs at least one z-plane per rank")
    comm.barrier()
    torch.cuda.synchronize()
    t_all = time.perf_counter()
    k1 = fus.complex_wavenumber(med, t.f0, 1)
    scale = fus.power_scale_factor(t, med, k1)
    res = SlabCascade(source_normalization=scale if scale > 0.0 else 1.0)
    g1 = grid_of(1)
    z0, nz = zsplit(g1.dims[2], G)[r]
    t0 = time.perf_counter()
    res.slabs.append(fus.evaluate_first_harmonic_zslab(t, med, g1, scale, z0, nz, ctx))
    torch.cuda.synchronize()
    p1_s = time.perf_counter() - t0
    res.grids.append(g1)
    res.slabs_z.append((z0, nz))
    for i in range(2, n + 1):
        gi = grid_of(i)
        ki = fus.complex_wavenumber(med, t.f0, i)
        z0, nz = zsplit(gi.dims[2], G)[r]
        t0 = time.perf_counter()
        lower = []
        for m in range(1, i):
            gm, pm = res.grids[m - 1], res.slabs[m - 1]
            if fus.same_grid(gm, gi):
                lower.append(_Vals(pm))
            elif cfg.recompute_p1_each_grid and m == 1:
                lower.append(_Vals(fus.evaluate_first_harmonic_zslab(t, med, gi, scale, z0, nz, ctx)))
            else:
                lo, planes = gather_source_planes(comm, gm, gi, pm)
                lower.append(_Vals(fus.interpolate_zslab(gm, planes, lo, gi, z0, nz, ctx)))
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        f = fus.rhs_source(i, lower, med, ki.omega, ctx)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        gk = fus.VoxelGrid(gi.lo, gi.hi, gi.dx, gi.dims, i)
        K = fus.SlabKernel(gk, ki, G, r, ctx)
        assert (K.z0, K.nz) == (z0, nz)
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        tr = transport
        if tr == "auto":
            px, py = fus.padded_dims(gk)[:2]
            warp = {256, 512, 768, 1024, 1536}  # lengths with transposing warp kernels
            tr = "p2p" if px in warp and py in warp else "nccl"
        if tr == "p2p":
            K.attach_peers(comm.all_gather_bytes(K.ipc_handles()))
            u = K.apply_p2p(f, -1.0)
        else:
            u = K.apply(f, -1.0)
        torch.cuda.synchronize()
        t4 = time.perf_counter()
        del K
        res.grids.append(gi)
        res.slabs.append(u)
        res.slabs_z.append((z0, nz))
        res.rows.append({"harmonic": i, "interpolate_s": comm.max(t1 - t0), "rhs_s": comm.max(t2 - t1),
                         "kernel_build_s": comm.max(t3 - t2), "apply_s": comm.max(t4 - t3),
                         "transport": tr, "p1_s": comm.max(p1_s) if i == 2 else 0.0})
    comm.barrier()
    torch.cuda.synchronize()
    res.solve_s = comm.max(time.perf_counter() - t_all)
    return res


class _Vals:  # rhs_source reads .values only
    def __init__(self, v):
        self.values = v
