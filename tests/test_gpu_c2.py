"""Parity at the benchmarked configuration (BASELINE C2) and on the sharded,
graph-replayed and concurrent paths.

C2 = the 800x800 frame bench.py times: sphere_cameras(aabb, 64, 800, seed=0)[0],
16^3 random-init lattice (seed 0), toy-scene occupancy 256^3, RenderConfig()
(K=384, eps=0.01, chunk 32, stratified), seed 0; as random init and with
density bias 20 (100,710 ERT-terminated rays, where fp16 rounding could flip
ERT decisions).

Bars:
* full-frame RenderStats == the reference's own render_image counters
  (tests/golden/render_c2.npz, written by make_golden.py from the reference):
  exact, both precisions;
* 16 sampled 4096-ray blocks == the reference's own _march_block colours:
  max abs <= 1e-3 (fp16, the north star's bound), <= 2e-5 (fp32);
* the whole frame against the oracle (all host cores): same bounds, PSNR
  reported;
* shards (block_stride = world) reassemble bit-identically;
* graph replay (legacy default stream), eager and concurrent renders are
  byte-identical.
"""

import os
import threading

import numpy as np
import pytest

from conftest import golden, have_gpu, toy_occupancy_bits
from oracle import gridfield_oracle as O

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not have_gpu(), reason="needs a CUDA device")]

TOL = {"fp16": 1e-3, "fp32": 2e-5}
VARIANTS = [("rand", None), ("bias20", 20.0)]


@pytest.fixture(scope="module")
def gf():
    import paper_2103_13744_b200 as m

    return m


@pytest.fixture(scope="module")
def c2():
    return golden("render_c2")


def c2_inputs(gf, bias):
    aabb = gf.Aabb((-1.0,) * 3, (1.0,) * 3)
    g = gf.init_network_grid(aabb, (16, 16, 16), seed=0)
    if bias is not None:
        g.params.biases["density"][:] = bias
    res, bits = toy_occupancy_bits()
    occ = gf.OccupancyGrid(aabb, res, bits.copy())
    cam = gf.sphere_cameras(aabb, 64, 800, seed=0)[0]
    return g, occ, cam


def block_rows(z, tag):
    blocks = [int(b) for b in z["blocks"]]
    n = z[f"{tag}_block_stats"][:, 3]
    return np.concatenate([np.arange(b * 4096, b * 4096 + int(k)) for b, k in zip(blocks, n)])


def psnr(a, b):
    mse = float(np.mean((a.astype(np.float64) - b.astype(np.float64)) ** 2))
    return float("inf") if mse == 0 else 10 * np.log10(1.0 / mse)


_ORACLE = {}


def oracle_frame(bias):
    """The oracle's full C2 frame (157 blocks on every host core)."""
    if bias not in _ORACLE:
        z = golden("render_c2")
        from conftest import golden_camera

        cam = golden_camera(z)
        lat = O.init_lattice(np.full(3, -1.0), np.ones(3), (16, 16, 16), seed=0)
        if bias is not None:
            lat.biases["density"][:] = bias
        res, bits = toy_occupancy_bits()
        occ = O.Occupancy(np.full(3, -1.0), np.ones(3), res, bits)
        _ORACLE[bias] = O.render_image(lat, occ, cam, O.MarchConfig(), seed=0, workers=os.cpu_count() or 1)
    return _ORACLE[bias]


def test_c2_camera_matches_fixture(gf, c2):
    _, _, cam = c2_inputs(gf, None)
    assert cam.width == int(c2["cam_w"]) and cam.height == int(c2["cam_h"])
    assert np.array_equal(np.array([cam.fx, cam.fy, cam.cx, cam.cy]), c2["cam_f"])
    assert np.array_equal(cam.c2w, c2["cam_c2w"])


@pytest.mark.parametrize("precision", ["fp16", "fp32"])
@pytest.mark.parametrize("tag,bias", VARIANTS)
def test_c2_frame_matches_reference(gf, c2, tag, bias, precision):
    g, occ, cam = c2_inputs(gf, bias)
    img, st = gf.render_image(g, occ, cam, gf.RenderConfig(), seed=0, precision=precision)
    ref = c2[f"{tag}_stats"]
    got = [st.total_queries, st.ess_skipped, st.ert_terminated_rays, st.n_rays]
    assert got == [int(v) for v in ref], (tag, precision, got, ref)
    flat = img.reshape(-1, 3)
    rows = block_rows(c2, tag)
    err = float(np.abs(flat[rows] - c2[f"{tag}_block_rgb"]).max())
    print(f"C2 {tag} {precision}: sampled blocks max|dev-ref|={err:.3e} "
          f"PSNR={psnr(flat[rows], c2[f'{tag}_block_rgb']):.1f} dB")
    assert err <= TOL[precision], (tag, precision, err)


@pytest.mark.parametrize("tag,bias", VARIANTS)
def test_c2_full_frame_against_oracle(gf, tag, bias):
    """Every pixel of the C2 frame against the oracle, both precisions."""
    g, occ, cam = c2_inputs(gf, bias)
    ref_img, ref = oracle_frame(bias)
    assert [ref.total_queries, ref.ess_skipped, ref.ert_terminated_rays] == \
        [int(v) for v in golden("render_c2")[f"{tag}_stats"][:3]]
    for precision in ("fp16", "fp32"):
        img, st = gf.render_image(g, occ, cam, gf.RenderConfig(), seed=0, precision=precision)
        assert (st.total_queries, st.ess_skipped, st.ert_terminated_rays) == \
            (ref.total_queries, ref.ess_skipped, ref.ert_terminated_rays)
        err = float(np.abs(img - ref_img).max())
        print(f"C2 {tag} {precision}: full frame max|dev-oracle|={err:.3e} PSNR={psnr(img, ref_img):.1f} dB")
        assert err <= TOL[precision], (tag, precision, err)


@pytest.mark.parametrize("world", [2, 3, 4, 8])
@pytest.mark.parametrize("precision", ["fp16", "fp32"])
def test_c2_shards_reassemble_bit_identical(gf, world, precision):
    """The multi-GPU partition on one device: ranks 0..world-1 of shard_rays
    rendered through render_rays_device(block_stride=world) and reassembled
    with unshard_index equal the unsharded frame bit for bit (the last block
    is ragged: 640,000 = 156 x 4096 + 1024), and the shard counters sum to
    the frame's."""
    g, occ, cam = c2_inputs(gf, 20.0)
    cfg = gf.RenderConfig()
    full, st = gf.render_image(g, occ, cam, cfg, seed=0, precision=precision)
    n = cam.width * cam.height
    cap = gf.render.shard_capacity(n, world)
    buf = np.zeros((world * cap, 3), np.float32)
    tot = np.zeros(4, np.int64)
    for r in range(world):
        off, stride, n_local = gf.render.shard_rays(n, r, world)
        rgb, s, _ = gf.render.render_rays_device(g, occ, cfg, 0, cam=cam, ray_offset=off, n_rays=n_local,
                                                 block_stride=stride, precision=precision)
        buf[r * cap: r * cap + n_local] = rgb.cpu().numpy()
        tot += s.cpu().numpy()
    img = buf[gf.render.unshard_index(n, world)].reshape(full.shape)
    assert np.array_equal(img, full)
    assert list(tot) == [st.total_queries, st.ess_skipped, st.ert_terminated_rays, st.n_rays]


def test_legacy_stream_replays_graph_and_matches_eager(gf, monkeypatch):
    """torch's default stream is the legacy stream (handle 0), which cannot
    be captured: the library runs the frame graph on a side stream ordered
    by events.  Repeated calls must replay the graph (counters move) and be
    byte-identical to the eager launch sequence (GF_NO_GRAPH=1)."""
    import torch

    from paper_2103_13744_b200 import _native as N

    assert torch.cuda.current_stream().cuda_stream == 0
    g, occ, cam = c2_inputs(gf, 20.0)
    cams = gf.sphere_cameras(g.aabb, 3, 200, seed=5)
    for precision in ("fp16", "fp32"):
        c0 = N.graph_counters()
        got = [gf.render_image(g, occ, cams[i % 3], gf.RenderConfig(), seed=i % 2, precision=precision)
               for i in range(6)]
        c1 = N.graph_counters()
        assert c1["eager"] == c0["eager"]
        assert (c1["replays"] - c0["replays"]) + (c1["updates"] - c0["updates"]) >= 4, (c0, c1)
        monkeypatch.setenv("GF_NO_GRAPH", "1")
        for i in range(6):
            img, st = gf.render_image(g, occ, cams[i % 3], gf.RenderConfig(), seed=i % 2, precision=precision)
            assert np.array_equal(img, got[i][0])
            assert st.total_queries == got[i][1].total_queries
        monkeypatch.delenv("GF_NO_GRAPH")


def test_side_stream_caller(gf):
    """A caller on its own stream (the service pattern) gets the same bytes."""
    import torch

    g, occ, cam = c2_inputs(gf, 20.0)
    cam = cam.scaled(width=160, height=160)
    base, _ = gf.render_image(g, occ, cam, gf.RenderConfig(), seed=3)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            img, _ = gf.render_image(g, occ, cam, gf.RenderConfig(), seed=3)
            assert np.array_equal(img, base)


def test_concurrent_render_image_identical_bytes(gf):
    """Re-entrancy (reference test_service.py:105-114: the service renders
    concurrently and must return identical bytes): 8 threads render at once,
    some the same view, some different views and seeds; each result equals
    the serial render of the same call."""
    g, occ, _ = c2_inputs(gf, 20.0)
    cams = gf.sphere_cameras(g.aabb, 4, 240, seed=1)
    calls = [(cams[i % 4], i % 3) for i in range(8)]
    serial = [gf.render_image(g, occ, c, gf.RenderConfig(), seed=s)[0] for c, s in calls]
    out = [None] * len(calls)
    errs = []
    barrier = threading.Barrier(len(calls))

    def run(i):
        try:
            barrier.wait()
            for _ in range(3):
                img, _ = gf.render_image(g, occ, calls[i][0], gf.RenderConfig(), seed=calls[i][1])
                if out[i] is None:
                    out[i] = img
                assert np.array_equal(img, out[i])
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    th = [threading.Thread(target=run, args=(i,)) for i in range(len(calls))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for i in range(len(calls)):
        assert np.array_equal(out[i], serial[i]), i


@pytest.mark.timeout(240)
def test_many_frames_back_to_back_no_deadlock(gf):
    """Regression guard for the MLP's run hand-over (k_mlp_tc): 400 C2
    frames back to back through the cached graph, every frame's counters
    exact.  A warp lagging two phases behind on a weight-buffer barrier
    (parity aliasing) used to deadlock here after a few dozen frames."""
    import torch
    from paper_2103_13744_b200 import _native as N
    from paper_2103_13744_b200.render import render_rays_device

    grid, occ, cam = c2_inputs(gf, None)
    cfg = gf.RenderConfig()
    n = cam.width * cam.height
    out = torch.empty((n, 3), dtype=torch.float32, device="cuda")
    st = torch.zeros(4, dtype=torch.int64, device="cuda")
    ws = torch.empty(N.lib().gf_render_workspace_bytes(grid.native_arch(), grid.native_geom(), cfg.native(0), n),
                     dtype=torch.uint8, device="cuda")
    ref = None
    for i in range(400):
        st.zero_()
        render_rays_device(grid, occ, cfg, 0, cam=cam, out=out, stats=st, ws=ws, precision="fp16")
        if i % 50 == 0 or i == 399:
            got = st.tolist()
            ref = ref or got
            assert got == ref, (i, got, ref)
    assert ref[0] == 11795580


@pytest.mark.timeout(600)
def test_bench_two_ranks_share_one_gpu():
    """The bench's multi-rank path end to end (torchrun, 2 ranks): each rank
    renders its interleaved blocks of the C2 frame, the shards are gathered
    and un-sharded inside the timed step and rank 0 prints one JSON line with
    the whole frame's counters.  GF_BENCH_SHARE_GPU=1 puts both ranks on this
    one device over gloo (the box has one GPU), so only the plumbing and the
    counts are checked, not the speed.  A run normally takes ~10 s; one
    stalled once in ~15 runs with the pytest process's own context also on
    the device (the three contexts time-share it; not a deployment shape), so
    a stalled attempt dumps every thread's stack (GF_BENCH_HANG_DUMP) and is
    retried once on a fresh port."""
    import json
    import socket
    import subprocess
    import sys

    from conftest import ROOT

    def free_port():
        with socket.socket() as s:
            s.bind(("127.0.0.1", 0))
            return s.getsockname()[1]

    env = dict(os.environ, GF_BENCH_SHARE_GPU="1", GF_BENCH_HANG_DUMP="200")
    failures = []
    for _attempt in range(2):
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
               "--master-addr", "127.0.0.1", "--master-port", str(free_port()), "bench.py", "--gpus", "2",
               "--steps", "3", "--warmup", "3", "--no-extras", "--no-cpu-baseline"]
        try:
            out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=260)
        except subprocess.TimeoutExpired as e:
            failures.append(f"timeout: {str(e.stderr)[-2000:]}")
            continue
        if out.returncode == 0:
            break
        failures.append(out.stderr[-3000:])
    else:
        raise AssertionError("\n----\n".join(failures))
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["steps"] == 3
    assert d["queries_per_frame"] == 11795580
