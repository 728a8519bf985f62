#!/usr/bin/env python3
"""Benchmark: one step = one pass of the whole hot path (EDT + LT + shell/reductions +
sphericity/roundness) over one synthetic label volume.

Default workload: BASELINE.json configs[3] (C4: 3D 1024^3 int32, ~20000 smooth + rough
grains, ~30 % fill) -- the 1024^3 volume the north-star target is quoted on; it fits one GPU.
With --gpus N > 1 (torchrun, one rank per GPU):
  * a 3D config (default C4) is split into N z-slabs of ONE volume: every step is one
    fastrs_sphericity_roundness_slab call with NCCL inside libfastrs (N8 halo z pass, or the
    N1 all-to-all transpose with --zpass transpose), "scaling": "strong";
  * C5 shards one seeded 256-image batch, rank r taking images [256r/N, 256(r+1)/N), no
    data-path collective, "scaling": "strong";
  * --mode volumes gives every rank its own volume ("scaling": "weak").

Timing: W warm-up steps, then K steps between barrier + cudaDeviceSynchronize, CUDA events
on the call's stream, max over ranks.  Inputs (4 GiB labels, ~16 GiB workspace) are larger
than the 126 MB L2, so no explicit flush is needed (stated in config).

--impl reference times the CPU oracle (the reference arm of this tier) on a bounded
sample of the same workload on the host cores (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Gvoxels/s end-to-end (EDT+LT+sphericity+roundness); % of HBM roofline"
UNIT = "Gvoxels/s"

# SURVEY.md §8(d) "Algorithmic bytes per element" (the roofline numerator): what
# the method must move with a multi-pass exact separable EDT on a grid larger than on-chip
# memory.  3D: K1 8, K2 8, K3 8, K4 4 (+8 per kept centre), K5 (dilate + shell + reduce) 5 =
# labels 4 + the shell flag 1; 2D: no K3.  K6 (per-label closed forms) is negligible.
ALG_BYTES_PER_ELEM = {"edt_x": 8.0, "edt_y": 8.0, "edt_z": 8.0, "prune": 4.0, "k5": 5.0, "metrics": 0.0}
ALG_BYTES_PER_KEPT = {"prune": 8.0}
# the library's per-stage CUDA events (fastrs_profile): K5 as §8(d) defines it is the candidate
# gather K5a + the paint with fused reductions K5b (+ the atomic fallback K5' and its
# reductions K5e, empty on the configs)
K5_PARTS = ("gather", "dilate", "epilogue")
# the kernels behind each stage (names in the ncu summaries under profiles/)
STAGE_KERNELS = {"edt_x": ["k_edt_x_seg", "k_edt_x"], "edt_y": ["k_edt_col16<0", "k_edt_col<0", "k_edt_col_fh<0"], "edt_z": ["k_edt_col16<1", "k_edt_col<1", "k_edt_col_fh<1"],
                 "prune": ["k_prune<1"], "k5": ["k_dilate_gather<1", "k_dilate_paint<1", "k_dilate_atomic<1",
                                               "k_epilogue_fallback<1"], "metrics": ["k_metrics"]}
STAGE_KERNELS_2D = dict(STAGE_KERNELS, edt_y=["k_edt_col16<1", "k_edt_col<1", "k_edt_col_fh<1"], prune=["k_prune<0"],
                        k5=["k_dilate_gather<0", "k_dilate_paint<0", "k_dilate_atomic<0", "k_epilogue_fallback<0"])
NCU_SUMMARY = os.path.join(ROOT, "profiles", "r02k_ncu_summary_c4.json")


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="fastrs", choices=["fastrs", "reference"])
    p.add_argument("--config", type=int, default=4, help="BASELINE.json config C1..C5 (default C4)")
    p.add_argument("--batch", type=int, default=None, help="C5 images per rank")
    p.add_argument("--e2e-steps", type=int, default=3)
    p.add_argument("--cpu-sample-slices", type=int, default=96,
                   help="CPU oracle sample: z-slices of the volume (3D) or images of the batch (2D)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--mode", default="auto", choices=["auto", "volumes", "slab"],
                   help="auto (default): N=1 the single-GPU call; N>1 a 3D config is split into z-slabs (one "
                        "volume, strong scaling, NCCL inside libfastrs) and C5 shards one seeded image batch "
                        "(strong scaling); volumes: an independent volume per rank (weak scaling); slab: the "
                        "z-slab path at any N")
    p.add_argument("--zpass", default="halo", choices=["halo", "transpose"],
                   help="slab z pass: h-slice halo (N8) or all-to-all z->y transpose (N1)")
    return p.parse_args()


def _kernel_key(name: str):
    """(base name, first template argument or None): 'k_prune<1, 1>' -> ('k_prune', '1')."""
    base, _, args = name.partition("<")
    return base.strip(), (args.split(",")[0].strip(" >") or None) if args else None


def ncu_record(kernel: str):
    """The committed ncu --set full summary line of `kernel` (dict), or None.  Names match on the
    base name and the first template argument (the 2D/3D instance), so a kernel that gained
    template parameters still finds its summary line."""
    try:
        kernels = json.load(open(NCU_SUMMARY))["kernels"]
    except Exception:
        return None
    k = kernels.get(kernel)
    if k is None:
        want = _kernel_key(kernel)
        for name, rec in kernels.items():
            got = _kernel_key(name)
            if got[0] == want[0] and (want[1] is None or got[1] == want[1]):
                k = rec
                break
    return k


def ncu_traffic(kernels) -> float | None:
    """DRAM bytes per launch summed over `kernels` (committed ncu summary), None if absent."""
    tot, found = 0.0, False
    for k in kernels:
        rec = ncu_record(k)
        if rec is not None:
            tot += rec["traffic_bytes_per_launch"]
            found = True
    return tot if found else None


def issue_roofline(per_stage_ms: dict, sm_mhz: float, n_sm: int, kernels=None) -> dict:
    """Instruction-issue roofline per stage: warp instructions per launch (committed ncu summary)
    / the live per-launch time, against 4 schedulers x 1 warp instruction per clock per SM at the
    SM clock sampled during the run.  The explanation of the HBM fractions: the kernels of this
    path are bound by instruction issue on data-dependent work, not by HBM bandwidth."""
    peak = n_sm * 4 * sm_mhz * 1e6
    out = {}
    for stage, ms in per_stage_ms.items():
        recs = [ncu_record(k) for k in (kernels or STAGE_KERNELS).get(stage, [])]
        wi = sum(r["warp_instructions"] or 0 for r in recs if r is not None)
        if ms <= 0 or not wi:
            continue
        ach = wi / (ms * 1e-3)
        out[stage] = {"achieved_winst_per_s": ach, "frac": round(ach / peak, 4)}
    return {"peak_winst_per_s": peak, "sm_mhz": sm_mhz, "sms": n_sm, "source": os.path.relpath(NCU_SUMMARY, ROOT),
            "stages": out}


def workload_name(cfg: int) -> str:
    return {1: "C1: 2D 256^2 int32, 20 ellipses + disc r=20",
            2: "C2: 3D 128^3 int32, 50 spheroids + sphere r=15",
            3: "C3: 3D 512^3 int32, 2000 smooth+rough grains, ~28% fill",
            4: "C4: 3D 1024^3 int32, ~20000 smooth+rough grains (r_eq power law 3-40), ~30% fill",
            5: "C5: batch of 2D 2048^2 int32 images, ~500 touching cells each"}[cfg]


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm = [float(r[1]) for r in self.rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) >= 9 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows if len(r) >= 9 for i in range(4) if r[5 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def make_input(cfg: int, batch, images=None):
    import synth
    t0 = time.time()
    lab, info = synth.make_config(cfg, batch=batch, images=images) if cfg == 5 else synth.make_config(cfg)
    info["gen_seconds"] = round(time.time() - t0, 1)
    ndim = 2 if cfg in (1, 5) else 3
    return lab, info, ndim


def oracle_sample(lab, ndim: int, slices: int):
    """The bounded CPU sample of a workload: a contiguous block of the volume (3D: `slices`
    z-slices from the middle; 2D batch: `slices` images) processed as its own grid."""
    if ndim == 3:
        z0 = max(0, (lab.shape[0] - slices) // 2)
        return np.ascontiguousarray(lab[z0:z0 + slices]), f"z-slab [{z0}, {z0 + slices}) of the volume"
    if lab.ndim == 3:
        return np.ascontiguousarray(lab[:slices]), f"images [0, {min(slices, lab.shape[0])}) of the batch"
    return lab, "the whole image"


def cpu_baseline(lab, info, ndim, slices: int) -> dict:
    """Time the oracle, as it stands, on the host cores on a bounded sample of the same workload
    (oracle_sample), processed as its own grid; value = sample elements / oracle wall time."""
    import oracle
    sub, where = oracle_sample(lab, ndim, slices)
    ml = info["max_label"]
    cores = os.cpu_count() or 1
    t0 = time.perf_counter()
    oracle.sphericity_roundness(sub, max_label=ml, ndim=ndim, nthreads=cores)
    dt = time.perf_counter() - t0
    n_obj = int(np.count_nonzero(np.bincount(sub.reshape(-1), minlength=ml + 1)[1:])) if sub.ndim == ndim else None
    return {"value": sub.size / dt / 1e9, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": (f"{where}: {sub.size} grid elements" + (f", {n_obj} objects" if n_obj is not None else "")
                       + f", run as its own grid (border background); value = elements / oracle wall time "
                       f"({dt:.2f} s on {cores} threads)"),
            "seconds": dt}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    lab, info, ndim = make_input(args.config, args.batch)
    vals = []
    for i in range(args.warmup + args.steps):
        cb = cpu_baseline(lab, info, ndim, args.cpu_sample_slices)
        if i >= args.warmup:
            vals.append(cb)
    v = statistics.mean(c["value"] for c in vals)
    sec = statistics.mean(c["seconds"] for c in vals)
    cb = dict(vals[-1])
    cb["value"] = v
    cb.pop("seconds", None)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u32/f64", "data": "synthetic",
            "config": {"workload": workload_name(args.config), "seed": info["seed"],
                       "elements": int(lab.size), "fill": round(info["fill"], 4)},
            "cpu_baseline": cb, "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0,
                                        "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_fastrs(args):
    import torch
    import torch.distributed as dist

    import paper_2504_05808_b200 as F

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    F.load()

    # C5 on N > 1 GPUs: rank r takes images [B*r/N, B*(r+1)/N) of one seeded B-image batch (strong
    # scaling, no data-path collective); otherwise every rank runs its own copy (weak scaling)
    shard = world > 1 and args.config == 5 and args.mode == "auto"
    b_total = args.batch or 256
    images = (b_total * rank // world, b_total * (rank + 1) // world) if shard else None
    lab, info, ndim = make_input(args.config, b_total if args.config == 5 else args.batch, images)
    ml = info["max_label"]
    B = lab.shape[0] if lab.ndim == ndim + 1 else 1
    M = B * ml
    t = torch.from_numpy(lab).to(dev)
    out = {"sphericity": torch.empty(M, dtype=torch.float64, device=dev),
           "roundness": torch.empty(M, dtype=torch.float64, device=dev)}
    ws = F.workspace(F.workspace_bytes(lab.shape, ndim, ml, F.HOST_IO), dev)
    stream = torch.cuda.current_stream(dev)

    def step():
        F.sphericity_roundness(t, max_label=ml, ndim=ndim, ws=ws, out=out)

    for _ in range(args.warmup):
        step()
    diag = F.diagnostics(ws)

    # ---- timed region -----------------------------------------------------------------
    clocks = ClockSampler(local)
    clocks.start()
    F.profile(True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        step()
    ev1.record(stream)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    stage_ms, calls = F.profile_read()
    F.profile(False)
    clk = clocks.stop()
    ms = ev0.elapsed_time(ev1) / args.steps
    ms_t = torch.tensor([ms], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    total_elems = b_total * lab.shape[-1] * lab.shape[-2] if shard else lab.size * world
    value = total_elems / (ms_max * 1e-3) / 1e9

    # ---- end to end through the host-buffer C entry point -------------------------------
    pinned = torch.from_numpy(lab).pin_memory()
    hs, hr = np.empty(M), np.empty(M)
    F.sphericity_roundness_host(pinned, max_label=ml, ndim=ndim, ws=ws, out=(hs, hr), device=dev)  # warm
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.e2e_steps):
        F.sphericity_roundness_host(pinned, max_label=ml, ndim=ndim, ws=ws, out=(hs, hr), device=dev)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    e2e_ms = torch.tensor([e0.elapsed_time(e1) / args.e2e_steps], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
    e2e_value = total_elems / (float(e2e_ms.item()) * 1e-3) / 1e9
    np.testing.assert_array_equal(hs, out["sphericity"].cpu().numpy())

    # ---- roofline (SURVEY.md §8(d) algorithmic bytes / live CUDA-event stage times) ----------
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "MEASURED_PEAKS.json hbm_gbs (copy bandwidth)" if "hbm_gbs" in peaks else "B200_PROFILING.md fallback"
    per = {k: v / max(calls, 1) for k, v in stage_ms.items()}  # ms per call and stage
    stage_ms_alg = {"edt_x": per["edt_x"], "edt_y": per["edt_y"], "prune": per["prune"], "metrics": per["metrics"],
                    "k5": sum(per[k] for k in K5_PARTS)}
    if ndim == 3:
        stage_ms_alg["edt_z"] = per["edt_z"]
    n = lab.size

    def alg_bytes(k):
        return ALG_BYTES_PER_ELEM[k] * n + ALG_BYTES_PER_KEPT.get(k, 0.0) * diag["n_kept"]

    SK = STAGE_KERNELS if ndim == 3 else STAGE_KERNELS_2D
    stages = {}
    for k, v in stage_ms_alg.items():
        gbs = alg_bytes(k) / (v * 1e-3) / 1e9 if v > 0 else 0.0
        stages[k] = {"ms": round(v, 4), "alg_bytes": alg_bytes(k), "GB/s": round(gbs, 1),
                     "frac": round(gbs / hbm_peak, 4), "kernels": SK[k]}
    dom = max((k for k in stage_ms_alg if k != "metrics"), key=lambda k: stage_ms_alg[k])
    dom_bytes = alg_bytes(dom)
    achieved = dom_bytes / (stage_ms_alg[dom] * 1e-3) / 1e9
    lt_bytes = alg_bytes("prune") + alg_bytes("k5")
    lt_ms = stage_ms_alg["prune"] + stage_ms_alg["k5"]
    path_bytes = sum(alg_bytes(k) for k in stage_ms_alg)
    path_gbs = path_bytes / (ms * 1e-3) / 1e9

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    cb = None
    if not args.no_cpu_baseline and world == 1:
        cb = cpu_baseline(lab, info, ndim, args.cpu_sample_slices)
        cb.pop("seconds", None)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True,
        # the N > 1 defaults split this same workload (C2-C4: z-slabs of the volume, C5: the one
        # 256-image batch), so N = 1 is the first point of a strong-scaling curve; --mode volumes
        # gives every rank its own volume (weak)
        "scaling": "strong" if (shard or (world == 1 and args.mode == "auto")) else "weak",
        "vs_baseline": None, "dtype": "u32/f64", "data": "synthetic",
        "config": {"workload": workload_name(args.config), "seed": info["seed"], "elements_per_gpu": int(n),
                   "fill": round(info["fill"], 4), "max_label": ml,
                   "parallelism": (f"images sharded over {world} GPUs ({b_total} total, rank 0: {images})" if shard
                                   else ("single GPU (N > 1 splits this volume into z-slabs / shards the batch)"
                                         if world == 1 and args.mode == "auto" else f"dp{world} (independent volumes)")),
                   "l2": "inputs larger than L2 (4 GiB labels + ~16 GiB workspace per step), no flush",
                   "input_sha256": info["sha256"], "input_hash_kind": info.get("sha256_kind")},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(lab.nbytes),
                "d2h_bytes_per_step": int(2 * M * 8), "ms_per_step": float(e2e_ms.item())},
        # K1 K2 (+fixup) K3 (+fixup) K4 K5a K5b K5' K5e K6 (3D); the 2D path has no K3
        # per call (ncu launch list of one call, profiles/r02k_ncu_summary_c4.json): K1; K2 (+ K3) as the 16-bit
        # scan, the slow-scan list and the envelope fix-up; K4; K5a + K5b in three waves with two wave resets;
        # K5', K5e (fallback tiles) and K6 -> 19 in 3D, 16 in 2D
        "gpu_launches": int((19 if ndim == 3 else 16) * args.steps),
        "roofline": {"bound": "hbm", "stage": dom, "kernels": SK[dom], "achieved": achieved,
                     "peak": hbm_peak, "unit": "GB/s", "frac": achieved / hbm_peak,
                     "traffic": ncu_traffic(SK[dom]),
                     "traffic_source": os.path.relpath(NCU_SUMMARY, ROOT), "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": dom_bytes, "ms_per_launch": stage_ms_alg[dom],
                     "bytes_rule": "SURVEY.md §8(d): K1 8, K2 8, K3 8, K4 4 + 8/kept centre, K5 5 B per grid element"},
        # the north-star number: local-thickness + reduction kernels (K4 + K5) against HBM
        "lt_reduction": {"stages": ["prune", "k5"], "ms": lt_ms, "alg_bytes": lt_bytes,
                         "GB/s": lt_bytes / (lt_ms * 1e-3) / 1e9,
                         "frac": lt_bytes / (lt_ms * 1e-3) / 1e9 / hbm_peak},
        "path": {"alg_bytes": path_bytes, "GB/s": path_gbs, "frac": path_gbs / hbm_peak},
        "stages": stages,
        "issue_roofline": issue_roofline(stage_ms_alg, float(clk.get("sm_mhz") or clk.get("sm_max_mhz") or 1965.0),
                                         torch.cuda.get_device_properties(dev).multi_processor_count, SK),
        "diagnostics": {k: int(v) for k, v in diag.items()},
        "clocks": clk,
        "cpu_baseline": cb,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_slab(args):
    """One volume split into z-slabs across the ranks: every step is one
    fastrs_sphericity_roundness_slab call (NCCL inside libfastrs: label halo, N8 halo or N1
    transpose z pass, D halo, allreduce of the partial sums).  Strong scaling: the whole
    volume's elements over the max-over-ranks time."""
    import torch
    import torch.distributed as dist

    import paper_2504_05808_b200 as F
    from paper_2504_05808_b200 import fastrs, slab

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    os.environ.setdefault("NCCL_DEBUG", "WARN")  # keep NCCL's banner off stdout (one JSON line)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    F.load()
    lab, info, ndim = make_input(args.config, args.batch)
    if ndim != 3:
        raise SystemExit("the z-slab path needs a 3D config")
    ml = info["max_label"]
    Z, Y, X = lab.shape
    slabs = fastrs.slab_partition(Z, world)
    z0, z1 = slabs[rank]
    host = torch.from_numpy(np.ascontiguousarray(lab[z0:z1])).pin_memory()
    del lab
    t = host.to(dev)
    comm = slab.make_comm()
    flags = fastrs.BORDER_BACKGROUND | (fastrs.SLAB_TRANSPOSE if args.zpass == "transpose" else 0)
    out = {"sphericity": torch.empty(ml, dtype=torch.float64, device=dev),
           "roundness": torch.empty(ml, dtype=torch.float64, device=dev)}
    res = {}

    def step():
        return fastrs.sphericity_roundness_slab(t, z0, Z, ml, comm, flags=flags, out=out)

    for _ in range(args.warmup):
        res = step()
    stream = torch.cuda.current_stream(dev)

    def timed(fn, k):
        dist.barrier()
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(k):
            fn()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        dist.barrier()
        m = torch.tensor([e0.elapsed_time(e1) / k], device=dev, dtype=torch.float64)
        dist.all_reduce(m, op=dist.ReduceOp.MAX)
        return float(m.item())

    clocks = ClockSampler(local)
    clocks.start()
    ms = timed(step, args.steps)
    clk = clocks.stop()
    hs, hr = torch.empty(ml, dtype=torch.float64).pin_memory(), torch.empty(ml, dtype=torch.float64).pin_memory()

    def e2e_step():  # the slab's labels from pinned host memory, results back to the host
        t.copy_(host, non_blocking=True)
        r = step()
        hs.copy_(r["sphericity"], non_blocking=True)
        hr.copy_(r["roundness"], non_blocking=True)

    e2e_ms = timed(e2e_step, args.e2e_steps)
    si = res.get("slab_info", {})
    xb = torch.tensor([si.get("bytes_sent", 0), si.get("bytes_received", 0)], device=dev, dtype=torch.int64)
    allx = [torch.zeros_like(xb) for _ in range(world)]
    dist.all_gather(allx, xb)
    n = Z * Y * X
    n_own = (z1 - z0) * Y * X
    value = n / (ms * 1e-3) / 1e9
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    # per-rank whole-path model: SURVEY.md §8(d) 33 B per own element (K1-K5), exchanges excluded
    path_gbs = 33.0 * n_own / (ms * 1e-3) / 1e9
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "u32/f64", "data": "synthetic",
                "config": {"workload": workload_name(args.config) + f", z-slabs over {world} GPU(s)",
                           "seed": info["seed"], "elements": int(n), "slabs": slabs, "parallelism": f"z-slab{world}",
                           "zpass": args.zpass + (" (N1 all-to-all transpose)" if args.zpass == "transpose"
                                                  else " (N8 h-slice halo)"),
                           "halo": {k: si.get(k) for k in ("mode", "h", "H", "dxy_max", "dmax", "halo_cap")},
                           "bytes_exchanged_per_rank": [{"sent": int(x[0]), "received": int(x[1])} for x in allx],
                           "l2": "inputs larger than L2, no flush"},
                "e2e": {"value": n / (e2e_ms * 1e-3) / 1e9, "unit": UNIT, "h2d_bytes_per_step": int(n * 4),
                        "d2h_bytes_per_step": int(2 * ml * 8 * world), "ms_per_step": e2e_ms},
                "gpu_launches": int(19 * args.steps),  # the single call's 19 (one rank; more z-pass ranges at N > 1)
                "roofline": {"bound": "hbm", "stage": "whole path per rank (K1-K6)", "achieved": path_gbs,
                             "peak": hbm_peak, "unit": "GB/s", "frac": path_gbs / hbm_peak, "traffic": None,
                             "bytes_rule": "SURVEY.md §8(d) 33 B per own grid element; exchanges not counted"},
                "clocks": clk, "cpu_baseline": None}
        print(json.dumps(line), flush=True)
    comm.close()
    dist.destroy_process_group()


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "reference":
        run_reference(args)
    elif args.mode == "slab" or (args.mode == "auto" and world > 1 and args.config in (2, 3, 4)):
        run_slab(args)
    else:
        run_fastrs(args)


if __name__ == "__main__":
    main()
