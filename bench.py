#!/usr/bin/env python
"""Benchmark of the KiloNeRF render hot path on B200 (BASELINE.json metric).

One step = one 800x800 frame per GPU (config C2: 16^3 grid of 32-wide tiny
MLPs, random init seed 0, toy-scene occupancy 256^3, K=384, eps=0.01,
ert_chunk=32), rendered through the device marcher; at N>1 every rank renders
its own view (sphere_cameras(aabb, 64, 800, seed=0)[rank], the C3 view batch)
and the images are all-gathered over NCCL inside the step.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--precision fp16|fp32]
  python bench.py --impl reference      # the reference's CPU algorithm (oracle port) on host cores

Prints ONE JSON line on rank 0.
"""

from __future__ import annotations

import os

# The CPU legs (reference arm, cpu_baseline) run numpy/OpenBLAS on a thread
# pool of host workers, as the reference's parallel_map does: one BLAS thread
# per worker.  OpenBLAS sizes its pool when numpy is first imported, so this
# must precede every numpy import (the GPU arm does no BLAS work).
for _v in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ[_v] = "1"

import argparse
import json
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "ms/frame and Mpixels/sec at 800x800, 16^3 tiny MLPs; MLP samples/sec vs roofline"
UNIT = "Mpix/s"
SIZE = 800
PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}
PAPER_1080TI_MPIX_S = 800 * 800 / 26e-3 / 1e6  # PAPER.md:166 (26 ms/frame, GTX 1080 Ti), context only


def workload_desc():
    """The C2 frame (identical for both arms; at N>1 the frame is split
    across the ranks by interleaved 4096-ray blocks and NCCL-gathered, C3)."""
    return {
        "workload": "C2: 800x800 frame, 16^3 grid of 32-wide tiny MLPs (random init, seed 0), toy-scene "
                    "occupancy 256^3 (tau=10, 10.81% occupied), K=384, eps=0.01, ert_chunk=32, stratified, seed 0",
        "image": [SIZE, SIZE], "grid": [16, 16, 16], "k": 384,
        "view": "sphere_cameras(aabb, 64, 800, seed=0)[0]",
        "multi_gpu": "N>1: the frame's 4096-ray blocks interleaved across ranks (shard_rays), NCCL all-gather of "
                     "the shards + unshard + 4-counter all-reduce inside the step (render_image_distributed)",
        "l2": "flushed between timed frames (256 MiB write outside the timed window)",
    }


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {k: float(d[k]) for k in ("hbm_gbs", "bf16_tflops", "bf16_tflops_sustained")}, "measured"
    return PEAKS_FALLBACK, "fallback"


def build_inputs(gf):
    aabb = gf.Aabb((-1.0,) * 3, (1.0,) * 3)
    grid = gf.init_network_grid(aabb, (16, 16, 16), seed=0)
    z = np.load(ROOT / "tests" / "golden" / "toy_occupancy_256.npz")
    occ = gf.OccupancyGrid(aabb, z["res"], z["bits"].copy())
    cams = gf.sphere_cameras(aabb, 64, SIZE, seed=0)
    return aabb, grid, occ, cams


def c4_desc(precision):
    return {
        "workload": "C4: 1920x1080 frame, 32^3 grid of 64-wide tiny MLPs (random init, seed 0), toy-scene occupancy "
                    "256^3, K=384, eps=0.01, ert_chunk=32, stratified, seed 0 (extra measurement, not the BASELINE line)",
        "image": [1920, 1080], "grid": [32, 32, 32], "width": 64, "k": 384, "mlp_precision": precision,
        "l2": "flushed between timed frames (256 MiB write outside the timed window)",
    }


def bulk_inputs(n, seed):
    """Reference bench.py:108-112 input recipe (BASELINE config 5): uniform
    float32 positions in [-1, 1]^3, normalised float32 normal directions."""
    rng = np.random.default_rng(seed)
    span = np.float32(2.0)
    pts = np.float32(-1.0) + rng.random((n, 3), dtype=np.float32) * span
    dirs = rng.normal(size=(n, 3)).astype(np.float32)
    dirs /= np.linalg.norm(dirs, axis=-1, keepdims=True)
    return pts, dirs


def run_bulk(args, rank, world, local):
    """Config 5: 2^26 random points/directions (reference bench.py:108-112
    recipe) through the 16^3 bank per step, no compositing.  Inputs resident
    in HBM for `value`; e2e copies them from pinned host memory every step."""
    import torch

    import paper_2103_13744_b200 as gf
    from paper_2103_13744_b200 import _native as N

    torch.cuda.set_device(local)
    n = 1 << 26
    grid = gf.init_network_grid(gf.Aabb((-1.0,) * 3, (1.0,) * 3), (16, 16, 16), seed=0)
    precision = args.precision or "fp16"
    grid.precision = precision
    pts, dirs = bulk_inputs(n, seed=1 + rank)
    p_h, d_h = torch.from_numpy(pts).pin_memory(), torch.from_numpy(dirs).pin_memory()
    p_d, d_d = p_h.cuda(), d_h.cuda()
    rgb_h = torch.empty((n, 3), dtype=torch.float32).pin_memory()
    sig_h = torch.empty((n,), dtype=torch.float32).pin_memory()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(args.warmup):
        grid.query_points(p_d, d_d)
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        # untimed pre-roll of the same load so nvidia-smi (first sample after
        # ~0.1 s) sees the clocks under load; the timed steps alone take ~30 ms
        t_end = time.perf_counter() + args.clock_preroll
        while time.perf_counter() < t_end:
            grid.query_points(p_d, d_d)
            torch.cuda.synchronize()
        launches0 = N.lib().gf_launch_count()
        for i in range(args.steps):
            flush.fill_(i & 0xFF)
            ev[i][0].record(stream)
            grid.query_points(p_d, d_d)
            ev[i][1].record(stream)
        torch.cuda.synchronize()
    launches = N.lib().gf_launch_count() - launches0
    ms = statistics.mean(a.elapsed_time(b) for a, b in ev)
    N.lib().gf_stage_timing(1)
    grid.query_points(p_d, d_d)
    torch.cuda.synchronize()
    st_ms, _ = N.stage_times()
    N.lib().gf_stage_timing(0)
    e2e_t = []
    for _ in range(max(3, args.steps // 2)):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        pd, dd = p_h.cuda(non_blocking=True), d_h.cuda(non_blocking=True)
        r, sg = grid.query_points(pd, dd)
        rgb_h.copy_(r, non_blocking=True)
        sig_h.copy_(sg, non_blocking=True)
        torch.cuda.synchronize()
        e2e_t.append(time.perf_counter() - t0)
    e2e_s = statistics.median(e2e_t)
    peaks, peak_src = load_peaks()
    flops = n * gf.count_flops(grid.arch)
    tf = flops / (st_ms["mlp"] * 1e-3) / 1e12
    line = {
        "metric": "MLP samples/sec vs roofline (config 5 bulk query)", "value": world * n / (ms * 1e-3) / 1e6,
        "unit": "Mquery/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f16" if precision == "fp16" else "f32",
        "data": "synthetic (reference bench.py recipe, random-init 16^3 lattice)",
        "config": {"workload": "C5: 2^26 random points/dirs through the 16^3 bank of 32-wide MLPs, no compositing",
                   "points": n, "l2": "flushed between timed steps; inputs 1.6 GB > L2"},
        "e2e": {"value": world * n / e2e_s / 1e6, "unit": "Mquery/s", "h2d_bytes_per_step": int(2 * pts.nbytes),
                "d2h_bytes_per_step": int(n * 16), "ms_per_step": e2e_s * 1e3},
        "roofline": {"bound": "tensor", "achieved": tf, "peak": peaks["bf16_tflops_sustained"], "unit": "TFLOP/s",
                     "frac": tf / peaks["bf16_tflops_sustained"], "traffic": None, "kernel": "mlp",
                     "peak_source": peak_src},
        "stage_ms": st_ms, "clocks": clk.summary(), "gpu_launches": int(launches),
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    return 0


def c4_camera(gf, aabb):
    """BASELINE config 4's 1920x1080 view: the focal length of
    sphere_cameras(aabb, 1, 1080, seed=0) on a 16:9 sensor."""
    c = gf.sphere_cameras(aabb, 1, 1080, seed=0)[0]
    return gf.Camera(1920, 1080, c.fx, c.fy, 960.0, 540.0, c.c2w)


def build_c4(gf):
    """Config 4: 32^3 lattice of 64-wide tiny MLPs (random init, seed 0), the
    toy-scene occupancy, one 1920x1080 view."""
    aabb = gf.Aabb((-1.0,) * 3, (1.0,) * 3)
    grid = gf.init_network_grid(aabb, (32, 32, 32), seed=0, arch=gf.MlpArchitecture(hidden_width=64))
    z = np.load(ROOT / "tests" / "golden" / "toy_occupancy_256.npz")
    occ = gf.OccupancyGrid(aabb, z["res"], z["bits"].copy())
    return aabb, grid, occ, c4_camera(gf, aabb)


# ---------------------------------------------------------------------------
# clocks during the timed region
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.sw_power_cap,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.rows = []
        self.proc = None
        self.thread = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:  # noqa: BLE001
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:  # noqa: BLE001
                self.proc.kill()
            self.thread.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ("sw_power_cap", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown")
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows),
                "window": "nvidia-smi every 100 ms over a pre-roll of the same load + the timed frames"}


# ---------------------------------------------------------------------------
# reference arm / CPU baseline: the oracle port of the reference algorithm
# ---------------------------------------------------------------------------
def cpu_render_sample(cam, block_stride: int, workers: int):
    """Render every `block_stride`-th 4096-ray block of the frame (1 = the
    whole frame) with the reference algorithm (oracle port of render.py:
    287-400, numpy, one OpenBLAS thread per worker as SURVEY §8d
    prescribes) on `workers` threads.  Returns (seconds, rays, queries)."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle import gridfield_oracle as O

    lat = O.init_lattice(np.full(3, -1.0), np.ones(3), (16, 16, 16), seed=0)
    z = np.load(ROOT / "tests" / "golden" / "toy_occupancy_256.npz")
    occ = O.Occupancy(np.full(3, -1.0), np.ones(3), z["res"], z["bits"])
    o, d = O.pixel_rays(cam.width, cam.height, cam.fx, cam.fy, cam.cx, cam.cy, cam.c2w)
    o64, d64 = o.astype(np.float64), d.astype(np.float64)
    starts = list(range(0, len(o), O.RAY_BLOCK))[::block_stride]
    cfg = O.MarchConfig()
    q = lambda p, dd: O.query_points(lat, p, dd)  # noqa: E731

    def one(s):
        gen = np.random.default_rng(np.random.SeedSequence([0, s]))
        e = min(s + O.RAY_BLOCK, len(o))
        _, _, ctr = O.march_block(q, lat.b_min, lat.b_max, occ, o64[s:e], d64[s:e], cfg, gen)
        return e - s, ctr.total_queries

    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=workers) as pool:
        res = list(pool.map(one, starts))
    dt = time.perf_counter() - t0
    return dt, sum(r[0] for r in res), sum(r[1] for r in res)


def cpu_workers():
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)


def run_reference(args, rank, world):
    """--impl reference: the reference's CPU algorithm (oracle port, pinned
    bit-identical to the reference by tests/test_oracle_golden.py) renders
    the WHOLE C2 frame (157 blocks) per step on every host core.  Warm-up
    steps render one block per worker (they only warm the thread pool and
    caches).  Timed steps stop early once --ref-budget-s is spent; `steps`
    then reports the frames actually timed."""
    if rank != 0:
        return 0
    import paper_2103_13744_b200 as gf

    _, _, _, cams = build_inputs(gf)
    workers = cpu_workers()
    n_blocks = (SIZE * SIZE + 4095) // 4096
    for _ in range(args.warmup):
        cpu_render_sample(cams[0], max(1, n_blocks // workers), workers)
    times, rays, t_start = [], 0, time.perf_counter()
    for _ in range(args.steps):
        dt, r, _ = cpu_render_sample(cams[0], 1, workers)
        times.append(dt)
        rays = r
        if time.perf_counter() - t_start > args.ref_budget_s:
            break
    ms = 1e3 * statistics.mean(times)
    mpix = rays / (ms * 1e-3) / 1e6
    sample = (f"the whole C2 frame per step ({rays} rays, {n_blocks} blocks of 4096), numpy oracle port of the "
              f"reference algorithm, {workers} worker threads x 1 OpenBLAS thread; {len(times)} timed frames")
    line = {
        "impl": "reference", "metric": METRIC, "value": mpix, "unit": UNIT, "n_gpus": world, "steps": len(times),
        "steps_requested": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64 sample placement / f32 MLP",
        "data": "synthetic", "config": workload_desc(),
        "cpu_baseline": {"value": mpix, "unit": UNIT, "cores": workers, "kind": "port", "sample": sample},
        "e2e": {"value": mpix, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def measure_extract(gf, torch, aabb, occ, reps=5):
    """the C2 occupancy bitmap (256^3 cells x 27 probes of the
    toy scene, tau=10) extracted on the device, CUDA-event timed, checked
    bit-for-bit against the reference's bitmap (tests/golden)."""
    sc = gf.standard_toy_scene()
    res = tuple(int(r) for r in occ.resolution)
    out = gf.extract_occupancy(sc.density_at, aabb, res, tau=10.0)  # warm-up
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    torch.cuda.synchronize()
    ev[0].record()
    for _ in range(reps):
        out = gf.extract_occupancy(sc.density_at, aabb, res, tau=10.0)
    ev[1].record()
    torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1]) / reps
    probes = 27 * int(np.prod(res))
    return {"ms": ms, "cells": int(np.prod(res)), "probes": probes, "gprobes_per_s": probes / ms / 1e6,
            "bit_exact_vs_reference": bool(np.array_equal(np.asarray(out.bits), np.asarray(occ.bits))),
            "note": "device extract_occupancy(standard_toy_scene().density_at, 256^3, tau=10) incl. the 2 MiB "
                    "bitmap D2H; the reference takes 6.7 s on 8 host cores for the same bitmap"}


def measure_train(gf, torch, aabb, occ, cam, reps=5, cpu=True):
    """one photometric training step at the reference's default
    batch (TrainConfig(): 8192 pixels of one 800x800 view, k_train=384, ESS on
    the toy occupancy, 16^3 random-init lattice): device time of the kernels
    (group + forward + loss + backward) by CUDA events, the step through the
    public API (photometric_loss_and_grads + adam_update, numpy parameters in
    and out as the reference's API requires), and the numpy oracle of the
    reference's math on the same batch (one host thread)."""
    from paper_2103_13744_b200 import train
    from paper_2103_13744_b200.batched import grouped_backward_device, grouped_forward_device

    grid = gf.init_network_grid(aabb, (16, 16, 16), seed=0)
    cfg = train.TrainConfig()
    o, d = gf.render.generate_rays(cam)
    rng = np.random.default_rng(0)
    pix = rng.choice(len(o), size=cfg.batch_size_pixels, replace=False)
    smp = train.prepare_ray_samples(o[pix], d[pix], aabb, cfg.k_train, True, rng, occ=occ)
    gt = rng.random((len(pix), 3)).astype(np.float32)
    q = len(smp.positions)
    state = train.AdamState.for_params(grid.params)
    for _ in range(2):  # warm-up: packing, workspaces, pinned host buffers
        _, grads = train.photometric_loss_and_grads(grid, smp, gt, cfg.background)
        train.adam_update(grid.params, grads, state, cfg.learning_rate, cfg)
    # kernels only: grouped forward + backward on device-resident rows
    layout = gf.group_by_network(gf.QueryBatch(smp.positions, smp.directions, grid.cell_index(smp.positions)),
                                 grid.n_cells)
    dc = torch.full((q, 3), 1e-3, device="cuda")
    ds = torch.full((q,), 1e-3, device="cuda")
    # device-resident grouped rows, as the training step has them (its batch
    # is grouped on the device): the timed forward is kernels only
    import dataclasses
    pos_g = torch.as_tensor(np.asarray(layout.positions, np.float32).reshape(-1, 3)).cuda()
    dir_g = torch.as_tensor(np.asarray(layout.directions, np.float32).reshape(-1, 3)).cuda()
    layout = dataclasses.replace(layout, offsets=torch.as_tensor(np.asarray(layout.offsets, np.int64)).cuda(),
                                 order=torch.as_tensor(np.asarray(layout.order, np.int64)).cuda())
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    cache = grouped_forward_device(grid, layout, pos_g, dir_g, keep_activations=True)
    for _ in range(2):  # allocator warm-up: the timed calls reuse cached blocks
        grouped_backward_device(grid, layout, cache, dc, ds)
    torch.cuda.synchronize()
    ev[0].record()
    for _ in range(reps):
        cache = grouped_forward_device(grid, layout, pos_g, dir_g, keep_activations=True)
    ev[1].record()
    for _ in range(reps):
        grouped_backward_device(grid, layout, cache, dc, ds)
    ev[2].record()
    torch.cuda.synchronize()
    fwd_ms, bwd_ms = ev[0].elapsed_time(ev[1]) / reps, ev[1].elapsed_time(ev[2]) / reps
    # one untimed API step first: the kernel timing above left other packed
    # weights and workspaces cached, and the first step re-validates them
    loss, grads = train.photometric_loss_and_grads(grid, smp, gt, cfg.background)
    train.adam_update(grid.params, grads, state, cfg.learning_rate, cfg)
    torch.cuda.synchronize()
    api = []
    for _ in range(reps):
        t0 = time.perf_counter()
        loss, grads = train.photometric_loss_and_grads(grid, smp, gt, cfg.background)
        train.adam_update(grid.params, grads, state, cfg.learning_rate, cfg)
        torch.cuda.synchronize()
        api.append(time.perf_counter() - t0)
    api_ms = statistics.median(api) * 1e3
    flop = 3 * 12392 * q  # forward + backward data + parameter gradients, count_flops units
    out = {"samples": q, "rays": len(pix), "k_train": cfg.k_train, "forward_kernel_ms": fwd_ms,
           "backward_kernel_ms": bwd_ms, "backward_tflops": flop * 2 / 3 / (bwd_ms * 1e-3) / 1e12,
           "api_step_ms": api_ms, "loss": loss,
           "note": "api_step_ms = median of 5 synchronised photometric_loss_and_grads + adam_update steps through the reference API (after one untimed step): the "
                   "gradients stay on the device unless read (DeviceGrads); the numpy parameters are updated in "
                   "place by one DMA into their page-locked storage; Adam moments stay on the device"}
    if cpu:
        from oracle import gridfield_oracle as O
        from oracle import train_oracle as T

        lat = O.lattice_from_grid(grid)
        t0 = time.perf_counter()
        T.photometric_loss_and_grads(lat, smp.positions, smp.directions, smp.ray_index, smp.slot, smp.deltas,
                                     smp.n_rays, smp.k, gt, cfg.background)
        out["cpu_oracle_s"] = time.perf_counter() - t0
        out["cpu_note"] = "numpy oracle of train.photometric_loss_and_grads on the same batch, 1 host thread"
    return out


def main():
    if os.environ.get("GF_BENCH_HANG_DUMP"):  # diagnostic: dump every thread's stack and exit if the run stalls
        import faulthandler

        faulthandler.dump_traceback_later(float(os.environ["GF_BENCH_HANG_DUMP"]), exit=True)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--precision", default=None, choices=[None, "fp16", "fp32"],
                    help="MLP precision (default: the library default render_image uses)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-budget-s", type=float, default=150.0,
                    help="reference arm: stop timing whole frames after this many seconds")
    ap.add_argument("--clock-preroll", type=float, default=0.6, help="seconds of untimed load before the timed frames")
    ap.add_argument("--no-extras", action="store_true", help="skip the extract / training side measurements")
    ap.add_argument("--workload", default="c2", choices=["c2", "c4", "c5"],
                    help="c2: the BASELINE metric's frame (default, the driver's line); c4: 32^3 lattice of "
                         "64-wide MLPs at 1920x1080; c5: 2^26-point bulk query (extra measurements)")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)
    if args.workload == "c5":
        return run_bulk(args, rank, world, local)

    import torch
    import torch.distributed as dist

    import paper_2103_13744_b200 as gf
    from paper_2103_13744_b200 import _native as N
    from paper_2103_13744_b200.render import ShardedFrame, render_image_distributed, render_rays_device

    # GF_BENCH_SHARE_GPU=1 (test only): several ranks on one device over gloo,
    # to exercise the multi-rank path (shards, gather, max-over-ranks timing)
    # on a single-GPU box; the numbers of such a run mean nothing
    share = os.environ.get("GF_BENCH_SHARE_GPU") == "1"
    if share:
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            if rank == 0:
                os.environ.setdefault("NCCL_DEBUG", "INFO")  # communicator log: N ranks, NVLS/P2P transport
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if args.workload == "c4":
        aabb, grid, occ, cam = build_c4(gf)
    else:
        aabb, grid, occ, cams = build_inputs(gf)
        cam = cams[0]
    n_pix = cam.width * cam.height
    cfg = gf.RenderConfig()
    if args.precision:
        grid.precision = args.precision
    precision = grid.resolved_precision(render=True)  # what render_image(grid, occ, cam, cfg) runs
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    frame = ShardedFrame(n_pix, rank, world, torch.device("cuda", local)) if world > 1 else None
    n_local = frame.n_local if frame else n_pix
    out = torch.empty((n_pix, 3), dtype=torch.float32, device="cuda") if frame is None else None
    stats = torch.zeros(4, dtype=torch.int64, device="cuda") if frame is None else frame.stats
    ws = torch.empty(N.lib().gf_render_workspace_bytes(grid.native_arch(), grid.native_geom(), cfg.native(0),
                                                       n_local), dtype=torch.uint8, device="cuda")

    def step():
        """One frame: the whole view at N=1; at N>1 this rank's interleaved
        blocks of the view, then the NCCL gather (render_image_distributed's
        device path with preallocated buffers)."""
        if frame is None:
            stats.zero_()
            render_rays_device(grid, occ, cfg, 0, cam=cam, out=out, stats=stats, ws=ws)
        else:
            render_image_distributed(grid, occ, cam, cfg, 0, frame=frame, ws=ws)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        os.environ["NCCL_DEBUG"] = "WARN"

    # ---- device-timed region (value)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    g0 = N.graph_counters()
    with ClockSampler(local) as clk:
        # pre-roll under the same load so nvidia-smi (>=100 ms period) has
        # samples spanning the timed window even when K frames take < 100 ms
        t_pre = time.perf_counter()
        while time.perf_counter() - t_pre < args.clock_preroll:
            step()
            torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        launches0 = N.lib().gf_launch_count()
        g0 = N.graph_counters()
        for i in range(args.steps):
            flush.fill_(i & 0xFF)
            ev[i][0].record(stream)
            step()
            ev[i][1].record(stream)
        torch.cuda.synchronize()
        launches = N.lib().gf_launch_count() - launches0
        g1 = N.graph_counters()
        if world > 1:
            dist.barrier()
    per = [a.elapsed_time(b) for a, b in ev]
    ms = sum(per) / len(per)
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = n_pix / (ms * 1e-3) / 1e6
    queries = int(stats[0].item())  # global after the gather at N>1
    graphs = {k: g1[k] - g0[k] for k in g1}

    # ---- stage breakdown + roofline (separate frames with stage events on;
    # this rank's share of the frame at N>1)
    N.lib().gf_stage_timing(1)
    n_prof = max(3, min(args.steps, 5))
    st_local = torch.zeros(4, dtype=torch.int64, device="cuda")
    for _ in range(n_prof):
        flush.fill_(1)
        st_local.zero_()
        if frame is None:
            render_rays_device(grid, occ, cfg, 0, cam=cam, out=out, stats=st_local, ws=ws)
        else:
            render_rays_device(grid, occ, cfg, 0, cam=cam, ray_offset=frame.offset, n_rays=frame.n_local,
                               block_stride=frame.stride, out=frame.local[: frame.n_local], stats=st_local, ws=ws)
    torch.cuda.synchronize()
    st_ms, st_n = N.stage_times()
    N.lib().gf_stage_timing(0)
    st_ms = {k: v / n_prof for k, v in st_ms.items()}
    st_n = {k: v // n_prof for k, v in st_n.items()}
    peaks, peak_src = load_peaks()
    flops_per_q = gf.count_flops(grid.arch)
    R, Q, rounds = n_local, int(st_local[0].item()), (cfg.k + cfg.ert_chunk - 1) // cfg.ert_chunk
    cell_bytes = 2 * grid.arch.parameter_count() if precision == "fp16" else 4 * grid.arch.parameter_count()
    algo = {  # SURVEY.md §8(d) per-unit figures x units per frame
        "mlp_flop": Q * flops_per_q,
        "mlp_bytes": Q * 36 + (791 if args.workload == "c2" else grid.n_cells) * cell_bytes,
        "march_bytes": Q * 40 + R * 12 + R * 16 * rounds + int(np.prod(occ.resolution)) // 8,
        "scatter_bytes": Q * 48,
    }
    mlp_tflops = algo["mlp_flop"] / (st_ms["mlp"] * 1e-3) / 1e12 if st_ms["mlp"] > 0 else 0.0
    march_gbs = algo["march_bytes"] / (st_ms["march"] * 1e-3) / 1e9 if st_ms["march"] > 0 else 0.0
    scatter_gbs = algo["scatter_bytes"] / (st_ms["scatter"] * 1e-3) / 1e9 if st_ms["scatter"] > 0 else 0.0
    # the frame's kernels run for ~1 ms at max clock: the burst tensor peak is
    # the denominator (the sustained figure is for seconds-long GEMM runs)
    peak_t = peaks["bf16_tflops"]
    stage_roof = {
        "mlp": {"bound": "tensor", "achieved": mlp_tflops, "peak": peak_t, "unit": "TFLOP/s",
                "frac": mlp_tflops / peak_t, "ms_per_frame": st_ms["mlp"], "launches_per_frame": st_n["mlp"]},
        "march": {"bound": "hbm", "achieved": march_gbs, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                  "frac": march_gbs / peaks["hbm_gbs"], "ms_per_frame": st_ms["march"],
                  "launches_per_frame": st_n["march"]},
        "scatter": {"bound": "hbm", "achieved": scatter_gbs, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                    "frac": scatter_gbs / peaks["hbm_gbs"], "ms_per_frame": st_ms["scatter"],
                    "launches_per_frame": st_n["scatter"]},
        "scan": {"ms_per_frame": st_ms["scan"], "launches_per_frame": st_n["scan"]},
        "setup": {"ms_per_frame": st_ms["setup"], "launches_per_frame": st_n["setup"]},
        "queries_this_rank": Q, "rays_this_rank": R,
    }
    dominant = max(("mlp", "march", "scatter"), key=lambda k: st_ms[k])
    traffic = None
    tfile = ROOT / "profiles" / "ncu_traffic.json"
    if tfile.exists() and world == 1:
        try:
            traffic = json.loads(tfile.read_text()).get(f"{args.workload}_{dominant}_{precision}")
        except Exception:  # noqa: BLE001
            traffic = None
    d = stage_roof[dominant]
    roofline = {"bound": d["bound"], "achieved": d["achieved"], "peak": d["peak"], "unit": d["unit"],
                "frac": d["frac"], "traffic": traffic, "kernel": dominant,
                "peak_source": f"{peak_src} ({'bf16_tflops burst' if d['bound'] == 'tensor' else 'hbm_gbs'})"}

    # ---- end-to-end through the public API (camera in, numpy image out)
    e2e_times = []
    for i in range(args.steps + 1):
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        if world == 1:
            img, st = gf.render_image(grid, occ, cam, cfg, seed=0)
        else:
            img_d, st = render_image_distributed(grid, occ, cam, cfg, seed=0)
            img = img_d.cpu().numpy() if rank == 0 else None
            torch.cuda.synchronize()
        if i:  # first call re-validates caches; not counted
            e2e_times.append(time.perf_counter() - t0)
    e2e_s = statistics.median(e2e_times)  # host jitter (pinned-block reuse, GIL) skews the mean
    if world > 1:
        t = torch.tensor([e2e_s], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e = {"value": n_pix / e2e_s / 1e6, "unit": UNIT,
           "h2d_bytes_per_step": int(N.C.sizeof(N.CameraT) + N.C.sizeof(N.MarchCfg)),
           "d2h_bytes_per_step": int(n_pix * 12 + 32), "ms_per_frame": e2e_s * 1e3,
           "api": "render_image(grid, occ, cam, RenderConfig(), seed=0)" if world == 1 else
                  "render_image_distributed(...) + image to host on rank 0"}
    if args.workload == "c2" and world == 1:
        # the C3 view batch through the same API, a different camera every frame
        # (each new view updates the cached frame graph in place)
        views = gf.sphere_cameras(aabb, 64, SIZE, seed=0)
        vt = []
        for v in views:
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            gf.render_image(grid, occ, v, cfg, seed=0)
            vt.append(time.perf_counter() - t0)
        e2e["views"] = {"n": len(vt), "median_ms_per_frame": statistics.median(vt) * 1e3,
                        "max_ms_per_frame": max(vt) * 1e3}

    extract = train_step = None
    if args.workload == "c2" and rank == 0 and world == 1 and not args.no_extras:
        extract = measure_extract(gf, torch, aabb, occ)
        train_step = measure_train(gf, torch, aabb, occ, cam, cpu=not args.no_cpu_baseline)

    # ---- CPU baseline (rank 0, N=1 only): the whole frame, all host cores
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and args.workload == "c2":
        workers = cpu_workers()
        dt, rays, _ = cpu_render_sample(cam, 1, workers)
        cpu = {"value": rays / dt / 1e6, "unit": UNIT, "cores": workers, "kind": "port",
               "sample": f"the whole C2 frame ({rays} rays), numpy oracle port of the reference algorithm, "
                         f"{workers} worker threads x 1 OpenBLAS thread, {dt:.1f} s"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong" if world > 1 else "weak",
            "vs_baseline": None, "dtype": "f16" if precision == "fp16" else "f32", "mlp_precision": precision,
            "data": "synthetic (random-init 16^3 lattice, analytic toy-scene occupancy)",
            "config": workload_desc() if args.workload == "c2" else c4_desc(precision),
            "e2e": e2e, "roofline": roofline, "cpu_baseline": cpu, "clocks": clk.summary(),
            "gpu_launches": int(launches), "graphs_in_timed_region": graphs,
            "queries_per_frame": queries, "mlp_samples_per_s": Q / (st_ms["mlp"] * 1e-3) if st_ms["mlp"] else None,
            "stage_roofline": stage_roof, "paper_1080ti_mpix_s_context": PAPER_1080TI_MPIX_S,
            "occupancy_extract": extract, "training_step": train_step,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
