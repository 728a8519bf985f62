"""Multi-GPU z-slab path: one large 3D volume split into z-slabs, one slab per rank
(BASELINE.json north_star "a single large volume is split into
z-slabs ... a halo exchange ... and an allreduce of per-label partial sums").

Every computation runs in the CUDA kernels behind the four slab phases of the C ABI
(include/fastrs.h "multi-GPU z-slab path"); this module only plans and performs the three
exchanges between them with torch.distributed (NCCL on GPUs; the CPU tests drive the same code
over gloo with a stand-in for the phases):

  A  edt_xy  (own slab)                       -> packed words, max D_xy
     1. allreduce(max) D_xy;  h = ceil(sqrt(max D_xy));  halo of h packed slices per side
  B  edt_z   (h-extended slab)                -> D of the own slab, max D
     2. allreduce(max) D;  H = isqrt(max D - 1) rounded up to a tile layer; halo of H D slices
  C  reduce  (H-extended slab; own tiles)     -> per-label u64 partial sums, u32 max LT^2
     3. allreduce(sum) partials, allreduce(max) max LT^2
  D  metrics                                  -> sphericity, roundness per label

Exactness: the z pass at an own element p only reads positions with
(p-q)^2 < D_xy(p) <= h^2; a kept ball that reaches the own slab has its centre within
isqrt(D-1) <= H slices; halo tiles may keep a few extra (redundant, still exact) centres
because their outer neighbours are missing; the partials are exact integers.  So the result is
bit-identical to the single-call path (tests/test_slab.py, tests/test_gpu_slab.py).
"""
from __future__ import annotations

import math

import torch
import torch.distributed as dist

ALIGN = 8            # slab boundaries fall on K4/K5 tile layers (tiles are 8 slices deep)
INF = (1 << 30) - 1  # "no site" partial distance (packed-word mask)


def partition(Z: int, nranks: int, align: int = ALIGN) -> list[tuple[int, int]]:
    """Split [0, Z) into nranks slabs whose inner boundaries are multiples of `align`."""
    bounds = [0]
    for i in range(1, nranks):
        b = int(round(Z * i / nranks / align)) * align
        bounds.append(min(max(b, bounds[-1]), Z))
    bounds.append(Z)
    slabs = [(bounds[i], bounds[i + 1]) for i in range(nranks)]
    if any(z1 <= z0 for z0, z1 in slabs):
        raise ValueError(f"cannot split Z={Z} into {nranks} non-empty slabs aligned to {align}")
    return slabs


def halo_edt(dxy_max: int, Z: int) -> int:
    """Slices the z pass needs on each side: the smallest h with h^2 >= max D_xy."""
    if dxy_max >= INF:
        return Z  # some element has no site in its x-y plane: the whole column matters
    return 0 if dxy_max <= 0 else math.isqrt(dxy_max - 1) + 1


def halo_lt(dmax: int, align: int = ALIGN) -> int:
    """Slices of D the dilation needs on each side: ball radius isqrt(D-1), rounded up to a
    whole tile layer so the extended slab stays tile aligned."""
    r = math.isqrt(dmax - 1) if dmax > 0 else 0
    return -(-r // align) * align


def halo_plan(slabs, w: int, Z: int):
    """Transfers that give every rank the `w` slices below and above its slab.
    Returns a list of (src, dst, side, a, b): global slices [a, b) go from src to dst's
    `side` ("lo" or "hi") halo buffer."""
    plan = []
    for dst, (z0, z1) in enumerate(slabs):
        for side, (a, b) in (("lo", (max(0, z0 - w), z0)), ("hi", (z1, min(Z, z1 + w)))):
            for src, (s0, s1) in enumerate(slabs):
                lo, hi = max(a, s0), min(b, s1)
                if src != dst and lo < hi:
                    plan.append((src, dst, side, lo, hi))
    return plan


def exchange_halo(own: torch.Tensor, slabs, rank: int, w: int, Z: int, group=None):
    """Collective: every rank receives the w slices below / above its slab from their owners.
    own: [nz, ...] tensor of this rank's slab.  Returns (lo, hi) tensors ([nlo, ...], [nhi, ...])."""
    z0, z1 = slabs[rank]
    lo = own.new_empty((z0 - max(0, z0 - w),) + tuple(own.shape[1:]))
    hi = own.new_empty((min(Z, z1 + w) - z1,) + tuple(own.shape[1:]))
    ops = []
    for src, dst, side, a, b in halo_plan(slabs, w, Z):
        if src == rank:
            s0 = slabs[src][0]
            ops.append(dist.P2POp(dist.isend, own[a - s0:b - s0].contiguous(), _peer(dst, group), group))
        elif dst == rank:
            buf, base = (lo, z0 - lo.shape[0]) if side == "lo" else (hi, z1)
            ops.append(dist.P2POp(dist.irecv, buf[a - base:b - base], _peer(src, group), group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    return lo, hi


def _peer(r: int, group):
    return r if group is None else dist.get_global_rank(group, r)


def _allreduce_max_int(v: torch.Tensor, group) -> int:
    t = v.reshape(-1)[:1].to(torch.int64).clone()
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return int(t.item())


class GpuPhases:
    """The four phases through the C ABI (argument marshalling only)."""

    def __init__(self):
        from . import fastrs
        self.F = fastrs

    def edt_xy(self, labels, below, max_label, flags):
        return self.F.slab_edt_xy(labels, below, max_label, flags)

    def edt_z(self, packed_ext, own_lo, own_hi, z_ext0, Z, flags):
        return self.F.slab_edt_z(packed_ext, own_lo, own_hi, z_ext0, Z, flags)

    def reduce(self, labels, d_ext, own_lo, own_hi, Z, dmax, max_label, flags):
        return self.F.slab_reduce(labels, d_ext, own_lo, own_hi, Z, dmax, max_label, flags)

    def metrics(self, part, nscale, dmax, stats):
        return self.F.metrics_from_partials(part, 3, nscale, dmax, stats=stats)

    def edge(self, labels, max_label, skip_zlo, skip_zhi):
        return self.F.touches_edge(labels, max_label, flags=(self.F.EDGE_SKIP_ZLO if skip_zlo else 0)
                                   | (self.F.EDGE_SKIP_ZHI if skip_zhi else 0))


def sphericity_roundness_slab(labels_slab: torch.Tensor, slabs, max_label: int, flags: int = 1, group=None,
                              phases=None, stats: bool = False) -> dict:
    """Collective over `group`: per-object sphericity/roundness of the volume whose z-slab
    `slabs[rank]` this rank holds in `labels_slab` ([nz][Y][X] int32).  Every rank returns
    the full per-label results (max_label entries).  `slabs` = partition(Z, world)."""
    phases = phases or GpuPhases()
    rank = dist.get_rank(group)
    Z = slabs[-1][1]
    z0, z1 = slabs[rank]
    nz, Y, X = labels_slab.shape
    if nz != z1 - z0:
        raise ValueError("labels_slab does not match slabs[rank]")
    info = {}
    # one collective before the first point-to-point batch: every rank joins the communicator
    chk = torch.tensor([nz], dtype=torch.int64, device=labels_slab.device)
    dist.all_reduce(chk, op=dist.ReduceOp.SUM, group=group)
    if int(chk.item()) != Z:
        raise ValueError("the ranks' slabs do not add up to the volume depth")
    # labels of the slice just below the slab (z-run flags of the first slice)
    lo_lab, _ = exchange_halo(labels_slab, slabs, rank, 1, Z, group)
    below = lo_lab[0] if lo_lab.shape[0] else None
    # A
    packed, dxy = phases.edt_xy(labels_slab, below, max_label, flags)
    h = halo_edt(_allreduce_max_int(dxy, group), Z)
    lo_p, hi_p = exchange_halo(packed, slabs, rank, h, Z, group)
    packed_ext = torch.cat([lo_p, packed, hi_p]) if (lo_p.shape[0] or hi_p.shape[0]) else packed
    # B
    d_own, dmax = phases.edt_z(packed_ext, lo_p.shape[0], lo_p.shape[0] + nz, z0 - lo_p.shape[0], Z, flags)
    dmax = _allreduce_max_int(dmax, group)
    H = halo_lt(dmax)
    lo_d, hi_d = exchange_halo(d_own, slabs, rank, H, Z, group)
    d_ext = torch.cat([lo_d, d_own, hi_d]) if (lo_d.shape[0] or hi_d.shape[0]) else d_own
    # C
    part = phases.reduce(labels_slab, d_ext, lo_d.shape[0], lo_d.shape[0] + nz, Z, dmax, max_label, flags)
    for k in ("vol", "n_shell", "sum_lt", "sum_shell_lt"):
        dist.all_reduce(part[k], op=dist.ReduceOp.SUM, group=group)
    dist.all_reduce(part["max_lt2"], op=dist.ReduceOp.MAX, group=group)
    # D
    res = phases.metrics(part, Z * Y * X, dmax, stats)
    info.update(h=h, H=H, dmax=dmax, halo_slices=int(lo_p.shape[0] + hi_p.shape[0] + lo_d.shape[0] + hi_d.shape[0]))
    res["slab_info"] = info
    return res


def touches_edge_slab(labels_slab: torch.Tensor, slabs, max_label: int, group=None, phases=None) -> torch.Tensor:
    """Collective: edge-object flags of the whole volume from z-slabs — every rank
    flags the labels on its slab's faces that are faces of the volume (its first / last slice
    only on the first / last rank), then allreduce(max).  Returns max_label uint8 flags."""
    phases = phases or GpuPhases()
    rank = dist.get_rank(group)
    z0, z1 = slabs[rank]
    Z = slabs[-1][1]
    f = phases.edge(labels_slab, max_label, z0 > 0, z1 < Z).to(torch.int32)
    dist.all_reduce(f, op=dist.ReduceOp.MAX, group=group)
    return f.to(torch.uint8)


def make_comm(group=None):
    """Collective over `group`: a libfastrs NCCL communicator (fastrs_comm_init) for
    fastrs.sphericity_roundness_slab.  Rank 0 draws the ncclUniqueId inside the library and
    torch.distributed broadcasts its 128 bytes (a CUDA tensor on an NCCL process group)."""
    from . import fastrs as F
    rank, n = dist.get_rank(group), dist.get_world_size(group)
    uid = F.nccl_unique_id() if rank == 0 else bytes(128)
    t = torch.tensor(list(uid), dtype=torch.uint8)
    if dist.get_backend(group) == "nccl":
        t = t.cuda()
    dist.broadcast(t, src=_peer(0, group), group=group)
    return F.Comm(bytes(t.cpu().tolist()), n, rank)


def simulate_slabs(labels: torch.Tensor, nranks: int, max_label: int, flags: int = 1, stats: bool = False,
                   phases=None, transpose: bool = False, lt_halo: str = "dense", split_zpass: bool = False) -> dict:
    """Single-process emulation of the slab path: the nranks slabs are processed one after
    another on one device and the exchanges become slicing of the assembled volume.  The
    same phases and halo widths as sphericity_roundness_slab; used by the GPU parity tests
    (one GPU here) to prove the phases bit-identical to the single-call path."""
    phases = phases or GpuPhases()
    Z, Y, X = labels.shape
    slabs = partition(Z, nranks)
    packed, dxy = [], 0
    for z0, z1 in slabs:
        below = labels[z0 - 1] if z0 > 0 else None
        p, d = phases.edt_xy(labels[z0:z1].contiguous(), below, max_label, flags)
        packed.append(p)
        dxy = max(dxy, int(d.reshape(-1)[0].item()))
    h = halo_edt(dxy, Z)
    packed = torch.cat(packed)
    dfull, dmax = [], 0
    if transpose:
        # N1: the z pass over whole columns of each rank's y-block (fastrs_sphericity_roundness_slab
        # with FASTRS_SLAB_TRANSPOSE), then back to the z-slab layout
        dvol = torch.empty_like(packed)
        for s_ in range(nranks):
            y0, y1 = Y * s_ // nranks, Y * (s_ + 1) // nranks
            if y1 > y0:
                d, m = phases.edt_z(packed[:, y0:y1].contiguous(), 0, Z, 0, Z, flags)
                dvol[:, y0:y1] = d
                dmax = max(dmax, int(m.reshape(-1)[0].item()))
        dfull = [dvol]
    else:
        for z0, z1 in slabs:
            a, b = max(0, z0 - h), min(Z, z1 + h)
            if split_zpass:
                # as the NCCL driver overlaps the halo exchange: the interior slices (>= h from a
                # face with a neighbour) first, then the two boundary ranges, each its own call
                i0, i1 = z0 + (h if z0 > 0 else 0), z1 - (h if z1 < Z else 0)
                rngs = [(i0, i1), (z0, i0), (i1, z1)] if i1 > i0 else [(z0, z1)]
                dd = torch.empty((z1 - z0,) + tuple(packed.shape[1:]), dtype=packed.dtype, device=packed.device)
                for r0, r1 in rngs:
                    if r1 > r0:
                        d, m = phases.edt_z(packed[a:b].contiguous(), r0 - a, r1 - a, a, Z, flags)
                        dd[r0 - z0:r1 - z0] = d
                        dmax = max(dmax, int(m.reshape(-1)[0].item()))
                dfull.append(dd)
                continue
            d, m = phases.edt_z(packed[a:b].contiguous(), z0 - a, z1 - a, a, Z, flags)
            dfull.append(d)
            dmax = max(dmax, int(m.reshape(-1)[0].item()))
    H = halo_lt(dmax)
    dfull = torch.cat(dfull)
    tot = None
    parts = []
    if lt_halo == "centres":
        # N4 (the in-library driver's default): each rank runs K4 on its own tile layers only
        # (D known 3 slices beyond its slab; the rest of its window is poisoned, so a read there
        # would show), then receives the K4 outputs of the layers within H slices from their owners
        from . import fastrs as F
        wins, wss = [], []
        for z0, z1 in slabs:
            a, b = max(0, z0 - H), min(Z, z1 + H)
            d = torch.full((b - a, Y, X), 0x3FFFFFFF, dtype=torch.int32, device=labels.device)
            lo, hi = max(a, z0 - 3), min(b, z1 + 3)
            d[lo - a:hi - a] = dfull[lo:hi]
            ws = F.workspace_for_slab((b - a, Y, X), labels.device)
            F.slab_prune(d, z0 - a, z1 - a, ws, flags)
            wins.append((a, b, d))
            wss.append(ws)
        recv_bytes = [0] * nranks
        for src, dst, side, a, b in halo_plan(slabs, H, Z):
            sa, da = wins[src][0], wins[dst][0]
            rec, ent = F.slab_pack_tiles(wss[src], wins[src][2].shape, (a - sa) // 8, (b - sa + 7) // 8)
            F.slab_unpack_tiles(wss[dst], wins[dst][2].shape, (a - da) // 8, (b - da + 7) // 8, rec, ent)
            recv_bytes[dst] += rec.numel() * 4 + ent.numel() * 8
        for src, dst, side, a, b in halo_plan(slabs, 3, Z):
            recv_bytes[dst] += (b - a) * Y * X * 4  # the 3-slice D halo of K4
        for r, (z0, z1) in enumerate(slabs):
            a, _, d = wins[r]
            parts.append(F.slab_dilate(labels[z0:z1].contiguous(), d, z0 - a, z1 - a, Z, dmax, max_label, wss[r], flags))
    else:
        for z0, z1 in slabs:
            a, b = max(0, z0 - H), min(Z, z1 + H)
            parts.append(phases.reduce(labels[z0:z1].contiguous(), dfull[a:b].contiguous(), z0 - a, z1 - a, Z, dmax,
                                       max_label, flags))
    for part in parts:
        if tot is None:
            tot = {k: v.clone() for k, v in part.items()}
        else:
            for k in ("vol", "n_shell", "sum_lt", "sum_shell_lt"):
                tot[k] += part[k]
            tot["max_lt2"] = torch.maximum(tot["max_lt2"], part["max_lt2"])
    res = phases.metrics(tot, Z * Y * X, dmax, stats)
    res["slab_info"] = dict(h=0 if transpose else h, H=H, dmax=dmax, slabs=slabs, transpose=transpose, lt_halo=lt_halo)
    # bytes each rank receives per exchange (what the NCCL driver moves for the same plan)
    yx4 = Y * X * 4
    zpass = [Z * (Y * (r + 1) // nranks - Y * r // nranks) * X * 4 - (z1 - z0) * (Y * (r + 1) // nranks - Y * r // nranks) * X * 4
             for r, (z0, z1) in enumerate(slabs)] if transpose else \
        [sum(b - a for s_, d_, _, a, b in halo_plan(slabs, h, Z) if d_ == r) * yx4 for r in range(nranks)]
    lt = recv_bytes if lt_halo == "centres" else \
        [sum(b - a for s_, d_, _, a, b in halo_plan(slabs, H, Z) if d_ == r) * yx4 for r in range(nranks)]
    res["slab_info"]["recv_bytes_zpass"] = zpass
    res["slab_info"]["recv_bytes_lt"] = lt
    return res
