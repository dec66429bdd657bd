#!/usr/bin/env python
"""Benchmark: solved frames/s of the LiveCap pose + non-rigid GN hot path.

Workload (BASELINE.json configs[2] shape, sharded per configs[4]): the full
two-stage per-frame solve (`solve_frame`: preprocessing, detection
conditioning, Stage I pose GN, Stage II non-rigid GN + PCG, snapping, warp)
on the x5k template (N=5,410) at 1024x1024, S independent synthetic capture
streams per GPU (seeds rank*S .. rank*S+S-1).  One step = one frame of every
stream.  Streams are independent, so ranks shard them with no collective on
the data path ("scaling": "weak"); only the timing barrier / max-reduce
touches torch.distributed.

  python bench.py [--gpus N --steps K --warmup W --streams S]
  python bench.py --impl reference      # the CPU implementation (oracle port)

`value` is measured with inputs resident in HBM (CUDA events on the library's
stream, max over ranks).  `e2e` is the same metric through the public
`Tracker` API from pinned host buffers: H2D of every step's images, masks and
detections and D2H of every step's poses + vertices are inside its timed
region.  Per-step inputs (S x ~100 MB of image + pyramid) exceed the 126 MB
L2, so no explicit flush is needed.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "solved frames/sec (pose+non-rigid GN) at 1/2/4/8 B200; PCG iter µs; % HBM BW"
DOMINANT = "k_surface_solve"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--streams", type=int, default=16, help="capture streams per GPU")
    ap.add_argument("--groups", type=int, default=4,
                    help="stream groups stepped concurrently on their own CUDA streams (BatchTracker)")
    ap.add_argument("--host-threads", type=int, default=1,
                    help="1: one host thread per group enqueues its step (BatchTracker host_threads)")
    ap.add_argument("--preset", default="x5k")
    ap.add_argument("--gn", type=int, default=None, help="non-rigid GN iterations (cfg4: 4)")
    ap.add_argument("--pcg", type=int, default=None, help="PCG iterations per GN step (cfg4: 8)")
    ap.add_argument("--res", type=int, default=1024)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e-u8", action="store_true", help="skip the 8-bit-frame e2e leg")
    ap.add_argument("--cpu-frames", type=int, default=3, help="timed steady frames of the CPU baseline")
    ap.add_argument("--directional", action="store_true",
                    help="SequenceConfig(directional=True): the reference's default, which loses the subject "
                         "on this workload (VERDICT r01); the default workload tracks (directional=False)")
    ap.add_argument("--no-quality", action="store_true", help="skip the untimed tracking-quality replay")
    ap.add_argument("--graph", action="store_true",
                    help="also time the CUDA-graph replay leg (opt-in: ncu's injection crashes on it)")
    ap.add_argument("--stage-pipeline", choices=["auto", "on", "off"], default="auto",
                    help="time the paper's pose -> non-rigid GPU-pair pipeline (StagePipeline) on cuda:0/cuda:1; "
                         "auto: when one process sees >= 2 devices")
    ap.add_argument("--dry-run", action="store_true",
                    help="multi-rank plumbing only (process group, sharding, max-over-ranks timing, gather); "
                         "no GPU, no solve - for CPU CI of the --gpus N path")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def shard_seeds(rank, streams_per_gpu):
    """Streams are independent TrackState recursions: rank r owns seeds
    r*S .. r*S+S-1 (no data-path collective)."""
    return [rank * streams_per_gpu + s for s in range(streams_per_gpu)]


def aggregate_fps(ms_per_rank, world, streams_per_gpu, steps):
    """Whole-job frames/s: every rank solved S frames per step; the job took
    as long as the slowest rank."""
    return world * streams_per_gpu * steps / (max(ms_per_rank) / 1e3)


def make_config(args):
    from paper_1810_02648_b200.config import SequenceConfig
    cfg = SequenceConfig(directional=bool(args.directional))
    if args.gn is not None:
        cfg.nonrigid.gn_iterations = args.gn
    if args.pcg is not None:
        cfg.nonrigid.pcg_iterations = args.pcg
    return cfg


def workload(args, world):
    return {"workload": f"cfg3-shaped full two-stage solve_frame, {args.preset} template @ "
                        f"{args.res}x{args.res}, {args.streams} synthetic streams per GPU (cfg5 sharding), "
                        f"{'directional' if args.directional else 'in-track (directional=False)'} silhouette rows",
            "preset": args.preset, "resolution": args.res, "streams_per_gpu": args.streams,
            "stream_groups": args.groups,
            "host_threads": bool(args.host_threads),
            "nonrigid_gn_pcg": [args.gn or 3, args.pcg or 4],
            "directional": bool(args.directional),
            "total_streams": args.streams * world, "parallelism": f"stream-sharded x{world}",
            "l2": "per-step inputs (images + pyramids) exceed the 126 MB L2; no flush needed"}


# ---------------------------------------------------------------------------
# synthetic inputs

def make_stream_frames(actor, cam, n_frames, seed, renderer, posing, device_rng=None):
    from paper_1810_02648_b200 import synthetic as S
    script = S.default_script(n_frames, noise=S.NoiseParams(sigma2d=1.0, sigma3d=0.008, seed=seed))
    return S.generate_sequence(actor, cam, script, renderer, posing, device_rng=device_rng)


def device_posing(ctx):
    from paper_1810_02648_b200.skinning import forward_kinematics, skin_points

    def posing(actor, pose, rest):
        fk = forward_kinematics(actor, pose, ctx=ctx)
        return skin_points(actor, pose, rest, ctx=ctx).positions, fk.positions, fk.marker_positions
    return posing


def device_renderer(ctx):
    from paper_1810_02648_b200.imageproc import render_attributes

    def render(cam, verts, tris, colors):
        return render_attributes(cam, verts, tris, colors, ctx=ctx)
    return render


# ---------------------------------------------------------------------------
# clocks during the timed region

class ClockSampler:
    def __init__(self, index):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={index}", f"--query-gpu={q}",
                                       "--format=csv,noheader,nounits", "-lms", "20"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.p = None
            return
        # nvidia-smi needs ~0.5 s to start; the timed region of a default run
        # is ~0.1 s, so wait until the sampler is live before it begins
        t0 = time.time()
        while time.time() - t0 < 10.0 and os.path.getsize(self.f.name) == 0 and self.p.poll() is None:
            time.sleep(0.02)

    def stop(self):
        if self.p is None:
            return None
        self.p.terminate()
        self.p.wait()
        self.f.seek(0)
        rows = [r.split(",") for r in self.f.read().strip().splitlines() if r.strip()]
        os.unlink(self.f.name)
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[1]))
                mx = max(mx, float(r[2]))
                for k, nm in enumerate(names):
                    if r[5 + k].strip().lower() == "active":
                        reasons.add(nm)
            except (ValueError, IndexError):
                continue
        if not sm:
            return None
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------
# algorithmic bytes of the Stage II kernel

def surface_bytes(N, E, delta):
    """delta = counter increments [frames, gn, pcg, trials, sumP, sumB, sumK, _]."""
    frames, gn, pcg, trials, sP, sB, sK = (float(v) for v in delta[:7])
    if frames == 0:
        return 0.0
    per_frame_img = 100.0 * sP + 21.0 * sB + 16.0 * sK      # summed over frames
    gn_per_frame = gn / frames
    trials_per_frame = trials / frames
    asm = gn * (192.0 * N + 88.0 * E) + gn_per_frame * per_frame_img
    pcg_b = pcg * (384.0 * N + 48.0 * E)
    trial = trials * (144.0 * N + 48.0 * E) + trials_per_frame * per_frame_img
    return asm + pcg_b + trial


def read_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def read_traffic():
    p = os.path.join(ROOT, "profiles", "ncu_surface_traffic.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d
    return None


# ---------------------------------------------------------------------------
# our arm

def run_ours(args):
    import numpy as np
    import torch

    rank, world, local = dist_env()
    # one process per GPU over NCCL.  BENCH_DIST_BACKEND=gloo exercises the
    # multi-rank path on fewer GPUs (ranks share devices round-robin)
    backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
    if backend != "nccl":
        local = local % max(torch.cuda.device_count(), 1)
    os.environ["LIVECAP_DEVICE"] = str(local)
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    coll_dev = f"cuda:{local}" if backend == "nccl" else "cpu"
    from paper_1810_02648_b200 import _lib
    from paper_1810_02648_b200 import synthetic as S
    from paper_1810_02648_b200.camera import suggest_camera
    from paper_1810_02648_b200.config import SequenceConfig
    from paper_1810_02648_b200.device import BatchTracker

    stream = torch.cuda.Stream(device=local, priority=-1)   # above the library's preprocessing stream
    ctx = _lib.Context(local, stream.cuda_stream)
    actor = S.build_actor(args.preset, with_skirt=True)
    cam = suggest_camera(args.res, args.res)
    Sn, K, W = args.streams, args.steps, args.warmup
    AHEAD = 2         # frames queued ahead of the one being solved (the library holds 3)
    F = W + K + AHEAD  # frames beyond the timed steps are queued, never solved
    t_gen = time.perf_counter()
    # inputs from the restated generator on the device: raster, skinning and
    # the numpy random stream (image noise, detections) all run on the GPU
    frames = [make_stream_frames(actor, cam, F, seed, device_renderer(ctx), device_posing(ctx), device_rng=ctx)
              for seed in shard_seeds(rank, Sn)]
    t_gen = time.perf_counter() - t_gen
    H, Wd = args.res, args.res
    # device-resident inputs for `value`
    img_d = torch.empty((Sn, F, H, Wd, 3), dtype=torch.float64, device=f"cuda:{local}")
    msk_d = torch.empty((Sn, F, H, Wd), dtype=torch.uint8, device=f"cuda:{local}")
    # pinned host inputs for `e2e`
    img_h = torch.empty((Sn, F, H, Wd, 3), dtype=torch.float64, pin_memory=True)
    msk_h = torch.empty((Sn, F, H, Wd), dtype=torch.uint8, pin_memory=True)
    for s in range(Sn):
        for f in range(F):
            img_h[s, f].copy_(torch.from_numpy(frames[s][f].image))
            msk_h[s, f].copy_(torch.from_numpy(frames[s][f].mask.astype(np.uint8)))
    img_d.copy_(img_h)
    msk_d.copy_(msk_h)
    torch.cuda.synchronize()
    dets = [[frames[s][f].detections for f in range(F)] for s in range(Sn)]
    cfg = make_config(args)

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        import torch.distributed as dist
        t = torch.tensor([x], dtype=torch.float64, device=coll_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- value: inputs resident in HBM.  Frames are queued ahead (the
    # reference's pipelined driver): step() solves frame f while the next
    # frame's preprocessing runs on the library's auxiliary stream.  Every
    # timed step queues one frame and solves one, so the timed region holds
    # exactly K solves and K preprocessings.  The S streams are split into
    # `groups` trackers stepped concurrently on their own CUDA streams; the
    # timed region is bracketed by device-wide synchronisations, so the
    # events measure the whole device.
    tr = BatchTracker(actor, cam, cfg, Sn, groups=args.groups, device=local,
                      host_threads=bool(args.host_threads))

    def queue_dev(f):
        for s in range(Sn):
            tr.set_frame(s, img_d[s, f].data_ptr(), msk_d[s, f].data_ptr(), dets[s][f], on_device=True)

    clocks = ClockSampler(local) if not os.environ.get("BENCH_NO_CLOCKS") else None
    # (sampling spans warm-up + the timed region)
    for f in range(AHEAD):
        queue_dev(f)
    for f in range(W):
        queue_dev(f + AHEAD)
        tr.step()
    tr.synchronize()
    c0 = [tr.counters(s) for s in range(Sn)]
    barrier()
    torch.cuda.synchronize()
    if not os.environ.get("BENCH_NO_PROFILE"):
        tr.profile_kernel(DOMINANT)
    l0 = tr.launches()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    host_q = host_s = 0.0
    for f in range(W, W + K):
        h0 = time.perf_counter()
        queue_dev(f + AHEAD)
        h1 = time.perf_counter()
        tr.step()
        host_s += time.perf_counter() - h1
        host_q += h1 - h0
    tr.synchronize()             # every group's solve, preprocessing and copy streams
    ev1.record(stream)
    ev1.synchronize()
    barrier()
    clk = clocks.stop() if clocks else None
    launches = tr.launches() - l0
    ms_dev = ev0.elapsed_time(ev1)
    k_ms, k_n = tr.profile_read()
    k_busy_ms = tr.profile_busy_ms()
    tr.profile_kernel(None)
    c1 = [tr.counters(s) for s in range(Sn)]
    ms_max = max_over_ranks(ms_dev)
    value = aggregate_fps([ms_max], world, Sn, K)
    # roofline of the dominant kernel
    N, E = actor.mesh.n_vertices, len(actor.mesh.edges)
    alg = sum(surface_bytes(N, E, c1[s] - c0[s]) for s in range(Sn))
    per_launch = alg / max(k_n, 1)
    k_avg_s = (k_ms / max(k_n, 1)) / 1e3
    peak, peak_src = read_peaks()
    achieved = per_launch / k_avg_s / 1e9 if k_avg_s > 0 else 0.0
    # the groups' launches run concurrently: all of the kernel's algorithmic
    # bytes over the union of its launch intervals
    achieved_agg = alg / (k_busy_ms / 1e3) / 1e9 if k_busy_ms > 0 else 0.0
    traffic = read_traffic()
    pcg_iters = sum(int((c1[s] - c0[s])[2]) for s in range(Sn))
    # µs per PCG iteration (the metric's second quantity): the PCG phases of
    # the last timed frame of every stream, from the solver's device
    # timestamps (%globaltimer; the groups run concurrently)
    pcg_us = []
    for s_ in range(Sn):
        _, sp = tr.phase_times(s_)
        for it in range(cfg.nonrigid.gn_iterations):
            a, b = sp[1 + 3 * it], sp[2 + 3 * it]
            if b > a > 0:
                pcg_us.append((b - a) / 1e3 / cfg.nonrigid.pcg_iterations)
    pcg_iter_us = float(np.median(pcg_us)) if pcg_us else None
    tr.close()

    # ---- the same device-resident loop with CUDA-graph replay of the
    # steady-state steps (lc_tracker_set_graph; no per-launch profiling, so it
    # is reported beside `value`, whose roofline needs the kernel events)
    graph_leg = None
    if args.graph:
        trg = BatchTracker(actor, cam, cfg, Sn, groups=args.groups, device=local,
                           host_threads=bool(args.host_threads))
        trg.set_graph(True)
        for f in range(AHEAD):
            for s in range(Sn):
                trg.set_frame(s, img_d[s, f].data_ptr(), msk_d[s, f].data_ptr(), dets[s][f], on_device=True)
        for f in range(W):
            for s in range(Sn):
                trg.set_frame(s, img_d[s, f + AHEAD].data_ptr(), msk_d[s, f + AHEAD].data_ptr(), dets[s][f + AHEAD],
                              on_device=True)
            trg.step()
        trg.synchronize()
        barrier()
        torch.cuda.synchronize()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        for f in range(W, W + K):
            for s in range(Sn):
                trg.set_frame(s, img_d[s, f + AHEAD].data_ptr(), msk_d[s, f + AHEAD].data_ptr(), dets[s][f + AHEAD],
                              on_device=True)
            trg.step()
        trg.synchronize()
        g1.record(stream)
        g1.synchronize()
        barrier()
        ms_g = max_over_ranks(g0.elapsed_time(g1))
        n_graphs, replays = trg.graph_stats()
        graph_leg = {"value": aggregate_fps([ms_g], world, Sn, K), "unit": "frames/s", "ms_per_step": ms_g / K,
                     "graphs": n_graphs, "replays": replays,
                     "how": "device-resident loop as `value`, steady-state steps replayed as captured CUDA "
                            "graphs (two per frame-queue phase and group: the auxiliary preprocessing branch and "
                            "the solve), no kernel profiling events; graphs bake buffer addresses, so each device "
                            "frame is first copied into the queue's own buffers (25 MB per stream-frame on the "
                            "copy engine) -- the device, not the host enqueue, bounds this loop, so the replay "
                            "does not pay for that copy"}
        trg.close()

    # ---- e2e: public API from pinned host buffers.  Frames are queued one
    # ahead as above (uploads overlap the solve) and every step's poses +
    # surfaces are read back into pinned host buffers with the streaming
    # readout; the host consumes frame f's results (event wait) while frame
    # f+1 is being solved (the pipelined driver's 2-slot latency).
    def run_e2e(imgs):
        tr2 = BatchTracker(actor, cam, cfg, Sn, groups=args.groups, device=local,
                           host_threads=bool(args.host_threads))
        x_h = torch.empty((2, Sn, 36), dtype=torch.float64, pin_memory=True)
        v_h = torch.empty((2, Sn, N, 3), dtype=torch.float64, pin_memory=True)
        done = [[torch.cuda.Event() for _ in tr2.ctxs] for _ in range(2)]
        checksum = [0.0]

        def queue_host(f):
            for s in range(Sn):
                tr2.set_frame(s, imgs[s, f].numpy(), msk_h[s, f].numpy(), dets[s][f])

        def step_host(f, first):
            tr2.step()
            b = f & 1
            for s in range(Sn):
                tr2.result_async(s, x_h[b, s], v_h[b, s])
            for ev, ts in zip(done[b], tr2.torch_streams):
                ev.record(ts)
            if not first:                     # frame f-1's results are complete on the host
                for ev in done[b ^ 1]:
                    ev.synchronize()
                checksum[0] += float(x_h[b ^ 1, :, 3].sum())

        for f in range(AHEAD):
            queue_host(f)
        for f in range(W):
            queue_host(f + AHEAD)
            step_host(f, f == 0)
        tr2.synchronize()
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for f in range(W, W + K):
            queue_host(f + AHEAD)
            step_host(f, False)
        for ev in done[(W + K - 1) & 1]:       # the last frame's results
            ev.synchronize()
        tr2.synchronize()
        e1.record(stream)
        e1.synchronize()
        barrier()
        return tr2, max_over_ranks(e0.elapsed_time(e1)), x_h, v_h

    tr2, ms_e2e, x_h, v_h = run_e2e(img_h)
    torch.cuda.set_device(local)
    # results of every stream to rank 0 (the tracking job's only collective,
    # NCCL; outside the timed regions): the last solved frame of each stream
    gathered = None
    if world > 1:
        from paper_1810_02648_b200.sharding import gather_results
        last = (W + K - 1) & 1
        g = gather_results(x_h[last][:, None].to(coll_dev), v_h[last][:, None].to(coll_dev),
                           world * Sn, "block")
        if rank == 0:
            gathered = int(g[0].shape[0])
    tr2.close()
    # ---- the paper's GPU-pair stage pipeline: Stage I on
    # cuda:0, Stage II on cuda:1, peer copies of poses / track state between
    # them; host frames as in e2e (mask-only upload to the pose device)
    pipe_line = None
    ndev = torch.cuda.device_count()
    if args.stage_pipeline == "on" or (args.stage_pipeline == "auto" and world == 1 and ndev >= 2):
        if ndev >= 2 and world == 1:
            try:   # (an informational leg: a failure here must not cost the bench line)
                pipe_line = run_stage_pipeline(actor, cam, cfg, Sn, img_h, msk_h, dets, W, K, AHEAD)
            except Exception as exc:  # noqa: BLE001
                pipe_line = {"error": f"{type(exc).__name__}: {exc}"[:300]}
        else:
            pipe_line = {"skipped": f"needs one process with two devices (devices {ndev}, ranks {world})"}
    # the same e2e loop with 8-bit frames (the reference's on-disk capture
    # format, frames/*.png read by load_color): the images are the synthetic
    # frames quantized to u8, converted on the device bit-exactly as
    # load_color does (u8 / 255); informational, the headline e2e stays f64
    e2e_u8 = None
    if not args.no_e2e_u8:
        img_q = torch.empty((Sn, F, H, Wd, 3), dtype=torch.uint8, pin_memory=True)
        for s_ in range(Sn):
            for f_ in range(F):
                img_q[s_, f_].copy_(torch.round(img_h[s_, f_] * 255.0).clamp_(0, 255).to(torch.uint8))
        tr3, ms_u8, _, _ = run_e2e(img_q)
        tr3.close()
        del img_q
        e2e_u8 = {"value": world * Sn * K / (ms_u8 / 1e3), "unit": "frames/s",
                  "h2d_bytes_per_step": Sn * (H * Wd * 3 + H * Wd + (actor.skeleton.n_joints + 4) * 2 * 8
                                              + actor.skeleton.n_joints * 3 * 8 + 2 * actor.skeleton.n_joints + 4),
                  "d2h_bytes_per_step": Sn * (36 * 8 + N * 3 * 8),
                  "note": "frames quantized to 8 bits (PNG capture format), uploaded as u8 and converted on the device"}
    # ---- tracking quality of the timed frames (untimed replay: the tracker
    # is deterministic, so the replay solves exactly the frames the timed
    # legs solved; checked against the e2e leg's last poses)
    quality = None
    if not args.no_quality:
        last = (W + K - 1) & 1
        quality = tracking_quality(actor, cam, cfg, Sn, args.groups, local, img_d, msk_d, dets, frames, W, K,
                                   x_h[last].numpy().copy())
    h2d = Sn * (H * Wd * 3 * 8 + H * Wd + (actor.skeleton.n_joints + 4) * 2 * 8
                + actor.skeleton.n_joints * 3 * 8 + 2 * actor.skeleton.n_joints + 4)
    d2h = Sn * (36 * 8 + N * 3 * 8)

    out = None
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            cpu = cpu_baseline(actor, cam, frames[0], args.cpu_frames, cfg)
        out = {
            "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world, "steps": K,
            "warmup": W, "ms_per_step": ms_max / K, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (reference generator restated)",
            "config": workload(args, world),
            "e2e": {"value": world * Sn * K / (ms_e2e / 1e3), "unit": "frames/s",
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
            "e2e_u8": e2e_u8,
            "graph": graph_leg,
            "stage_pipeline": pipe_line,
            "gpu_launches": launches,
            "roofline": {"bound": "hbm", "kernel": DOMINANT, "achieved": achieved, "peak": peak,
                         "unit": "GB/s", "frac": achieved / peak if peak else None,
                         # ncu DRAM bytes of one launch, scaled from the captured
                         # launch's stream count to this run's streams per launch
                         "traffic": (traffic["dram_bytes_per_launch"] * (Sn / max(args.groups, 1))
                                     / traffic["streams"] if traffic and traffic.get("streams") else None),
                         "algorithmic_bytes_per_launch": per_launch,
                         "kernel_ms_per_launch": k_avg_s * 1e3, "launches": k_n,
                         "achieved_concurrent": achieved_agg,
                         "frac_concurrent": achieved_agg / peak if peak else None,
                         "kernel_busy_ms": k_busy_ms,
                         "note": ("achieved/frac: per launch (one launch = one group of "
                                  f"{args.streams // max(args.groups, 1)} streams); *_concurrent: every launch's "
                                  "algorithmic bytes over the union of the launch intervals of all groups"),
                         "peak_source": peak_src,
                         "traffic_source": (traffic or {}).get("source")},
            "pcg_iterations_timed": pcg_iters,
            "pcg_iter_us": pcg_iter_us,
            "pcg_iter_us_note": "median over the last timed frame's GN steps of every stream of "
                                "(PCG phase incl. setup) / iterations, device timestamps",
            "gathered_streams": gathered,
            "per_stream_fps": 1e3 * K / ms_max,
            # host wall time per step spent queueing frames / enqueueing the
            # groups' steps (close to ms_per_step = host-bound enqueue)
            "host_ms_per_step": {"queue": 1e3 * host_q / K, "step": 1e3 * host_s / K},
            "clocks": clk,
            "tracking": quality,
            "cpu_baseline": cpu,
            "input_generation_s": round(t_gen, 2),
        }
        print(json.dumps(out))
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return out


# ---------------------------------------------------------------------------
# GPU-pair stage pipeline leg

def run_stage_pipeline(actor, cam, cfg, Sn, img_h, msk_h, dets, W, K, AHEAD):
    """frames/s of device.StagePipeline (pose device 0, surface device 1):
    host frames queued AHEAD frames ahead, K timed steps after W warm-up
    steps; timed with CUDA events on both devices (the max of the two)."""
    import numpy as np
    import torch

    from paper_1810_02648_b200.device import StagePipeline
    groups = 2 if Sn % 2 == 0 else 1
    pipe = StagePipeline(actor, cam, cfg, Sn, pose_device=0, surface_device=1, groups=groups)

    def queue(f):
        for s in range(Sn):
            pipe.set_frame(s, img_h[s, f].numpy(), msk_h[s, f].numpy(), dets[s][f])

    for f in range(AHEAD):
        queue(f)
    for f in range(W):
        queue(f + AHEAD)
        pipe.step()
    pipe.synchronize()
    evs = []
    for d in (0, 1):
        with torch.cuda.device(d):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            evs.append((d, e0, e1))
    for f in range(W, W + K):
        queue(f + AHEAD)
        pipe.step()
    pipe.synchronize()
    ms = 0.0
    for d, e0, e1 in evs:
        with torch.cuda.device(d):
            e1.record()
            e1.synchronize()
            ms = max(ms, e0.elapsed_time(e1))
    x_last = [pipe.result(s, with_report=False)[0] for s in range(Sn)]
    pipe.close()
    return {"value": Sn * K / (ms / 1e3), "unit": "frames/s", "devices": [0, 1], "stream_groups": groups,
            "ms_per_step": ms / K, "finite": bool(all(bool(np.isfinite(x).all()) for x in x_last)),
            "how": "StagePipeline: Stage I (conditioning + pose GN) on cuda:0, Stage II (surface GN, PCG, "
                   "snapping) on cuda:1; per frame cudaMemcpyPeerAsync of the poses (0 -> 1) and the "
                   "Stage-I track state (1 -> 0); host frames (mask-only to cuda:0)"}


# ---------------------------------------------------------------------------
# tracking quality of the timed frames (metrics.py / evaluation.py on the device)

def tracking_quality(actor, cam, cfg, Sn, groups, local, img_d, msk_d, dets, frames, W, K, x_last_e2e):
    import numpy as np

    from paper_1810_02648_b200.device import BatchTracker
    from paper_1810_02648_b200.imageproc import render_mask
    from paper_1810_02648_b200.metrics import aligned_joint_error_batch, iou_batch, mean_vertex_error_batch
    from paper_1810_02648_b200.skinning import forward_kinematics

    tr = BatchTracker(actor, cam, cfg, Sn, groups=groups, device=local, host_threads=False)
    N = actor.mesh.n_vertices
    V = np.empty((Sn, K, N, 3))
    X = np.empty((Sn, K, 36))
    for f in range(W + K):
        for s in range(Sn):
            tr.set_frame(s, img_d[s, f].data_ptr(), msk_d[s, f].data_ptr(), dets[s][f], on_device=True)
        tr.step()
        if f >= W:
            for s in range(Sn):
                x, v, _, _ = tr.result(s, with_report=False)
                X[s, f - W], V[s, f - W] = x, v
    tr.close()
    ious, verr, jerr = [], [], []
    for s in range(Sn):
        fr = frames[s][W:W + K]
        verr.append(mean_vertex_error_batch(V[s], np.stack([q.gt_vertices for q in fr])))
        joints = np.stack([forward_kinematics(actor, X[s, k]).positions for k in range(K)])
        jerr.append(aligned_joint_error_batch(joints, np.stack([q.gt_joints for q in fr])))
        masks = np.stack([render_mask(cam, V[s, k], actor.mesh.triangles) for k in range(K)])
        ious.append(iou_batch(masks, np.stack([q.mask for q in fr])))
    ious, verr, jerr = np.array(ious), np.array(verr), np.array(jerr)
    per_stream = ious.mean(axis=1)
    return {"frames": [W, W + K - 1], "streams": Sn,
            "iou_mean": float(ious.mean()), "iou_min": float(ious.min()),
            "iou_per_stream": [round(float(v), 4) for v in per_stream],
            "streams_iou_ge_0_9": int((per_stream >= 0.9).sum()),
            "vertex_error_mm_mean": 1e3 * float(verr.mean()), "vertex_error_mm_max": 1e3 * float(verr.max()),
            "aligned_joint_error_mm_mean": 1e3 * float(jerr.mean()),
            "replay_identical": bool(np.array_equal(X[:, K - 1], x_last_e2e)),
            "how": "untimed replay of the timed frames through the public API; silhouette IoU of the "
                   "solved surface vs the observed mask, centred mean vertex error vs ground truth, "
                   "Procrustes-aligned joint error (metrics.py, on the device)"}


# ---------------------------------------------------------------------------
# CPU baseline: the oracle (a restatement of the reference, bit-identical to
# it) timed on one host core on a bounded sample of the same workload

def cpu_baseline(actor, cam, frames, n_timed, cfg):
    from threadpoolctl import threadpool_limits

    from oracle import frame as OF
    with threadpool_limits(1):
        st = OF.State()
        # untimed cold start (frame 0), then n_timed steady frames end to end
        prep = OF.prepare(frames[0].image, frames[0].mask, frames[0].detections, actor, cfg)
        _, _, _, st, _, _ = OF.solve_frame(prep, actor, cam, cfg, st)
        t0 = time.perf_counter()
        n = 0
        for fr in frames[1:1 + n_timed]:
            prep = OF.prepare(fr.image, fr.mask, fr.detections, actor, cfg)
            _, _, _, st, _, _ = OF.solve_frame(prep, actor, cam, cfg, st)
            n += 1
        dt = time.perf_counter() - t0
        # the PCG alone: the next frame's first Stage II system
        # in the reference's explicit block layout, pcg_solve best of 5
        from oracle import linsolve as OL, surface as OSF
        fr = frames[min(1 + n_timed, len(frames) - 1)]
        prep = OF.prepare(fr.image, fr.mask, fr.detections, actor, cfg)
        drest = actor.mesh.rest_vertices + st.disp_rest
        x, _ = OF.stage1(prep, actor, cam, cfg, st, drest)
        pb, v_init, _, _ = OF.stage2_problem(prep, actor, cam, cfg, st, x, drest)
        system = OSF.normal_system(pb, OSF.surface_evaluate(pb, v_init, 0))
        iters = cfg.nonrigid.pcg_iterations
        best = float("inf")
        for _ in range(5):
            p0 = time.perf_counter()
            OL.pcg(*system, iterations=iters)
            best = min(best, time.perf_counter() - p0)
    return {"value": n / dt, "unit": "frames/s", "cores": 1, "kind": "port",
            "sample": f"1 stream, {n} steady frames (after an untimed frame 0), preprocess + solve_frame, "
                      f"1 thread, oracle port of the reference (bit-identical outputs)",
            "pcg_iter_us": 1e6 * best / iters,
            "pcg_note": f"pcg_solve on one Stage II system (N={actor.mesh.n_vertices}, explicit block layout), "
                        f"{iters} iterations, best of 5, 1 thread"}


# ---------------------------------------------------------------------------
# reference arm: the reference's CPU implementation (oracle port) on all host
# cores, one process per stream

def _ref_worker(a):
    preset, res, n_frames, seed, warm, gn, pcg, directional = a
    os.environ["OMP_NUM_THREADS"] = "1"
    from threadpoolctl import threadpool_limits

    from oracle import frame as OF
    from oracle import geometry as OG
    from oracle import imaging as OI
    from paper_1810_02648_b200 import synthetic as S
    from paper_1810_02648_b200.camera import suggest_camera
    from paper_1810_02648_b200.config import SequenceConfig

    def posing(actor, pose, rest):
        fk = OG.Fk(actor.skeleton, pose.to_vector())
        return OG.skin(rest, actor.skinning, fk.dqs)[0], fk.pos, fk.markers

    actor = S.build_actor(preset, with_skirt=True)
    cam = suggest_camera(res, res)
    frames = make_stream_frames(actor, cam, n_frames, seed, OI.render_attributes, posing)
    cfg = SequenceConfig(directional=directional)
    if gn is not None:
        cfg.nonrigid.gn_iterations = gn
    if pcg is not None:
        cfg.nonrigid.pcg_iterations = pcg
    st = OF.State()
    stamps = []
    with threadpool_limits(1):
        for fr in frames:
            prep = OF.prepare(fr.image, fr.mask, fr.detections, actor, cfg)
            _, _, _, st, _, _ = OF.solve_frame(prep, actor, cam, cfg, st)
            stamps.append(time.perf_counter())
    return stamps[warm - 1], stamps[-1], len(frames) - warm


def run_reference(args):
    import multiprocessing as mp
    rank, world, _ = dist_env()
    if rank != 0:
        return None
    cores = len(os.sched_getaffinity(0))
    procs = max(1, min(args.streams, cores))
    W = max(1, args.warmup)
    K = max(1, args.steps)
    jobs = [(args.preset, args.res, W + K, s, W, args.gn, args.pcg, bool(args.directional)) for s in range(procs)]
    with mp.get_context("fork").Pool(procs) as pool:
        res = pool.map(_ref_worker, jobs)
    spans = [b - a for a, b, _ in res]
    frames = sum(n for _, _, n in res)
    value = frames / max(spans)
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world,
           "steps": K, "warmup": W, "ms_per_step": 1e3 * max(spans) / K, "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (reference generator restated)",
           "config": workload(args, world),
           "cpu_baseline": {"value": value, "unit": "frames/s", "cores": procs, "kind": "port",
                            "sample": f"{procs} streams in parallel processes (1 thread each), {K} steady "
                                      f"frames per stream after {W} untimed, preprocess + solve_frame"},
           "e2e": {"value": value, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))
    return out


def spawn_ranks(args):
    """`bench.py --gpus N` without a torchrun environment: launch N ranks
    (one process per GPU) the way the driver does and pass rank 0's line
    through."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.run(cmd).returncode


def run_dry(args):
    """--dry-run: the multi-rank plumbing of run_ours without a GPU (CPU CI):
    process group, stream sharding, barrier, max-over-ranks time, result
    gather to rank 0, rank-0 JSON line.  No solve runs; the line says so."""
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_1810_02648_b200.sharding import assign_streams, gather_results
    rank, world, _ = dist_env()
    if world > 1:
        dist.init_process_group("gloo")
    Sn, K = args.streams, args.steps
    mine = assign_streams(Sn * world, world, rank, "block")
    assert mine == shard_seeds(rank, Sn)
    t0 = time.perf_counter()
    time.sleep(0.01 * (rank + 1))
    ms = 1e3 * (time.perf_counter() - t0)
    if world > 1:
        dist.barrier()
        t = torch.tensor([ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        poses = np.stack([np.full((1, 36), float(s)) for s in mine])
        verts = np.stack([np.full((1, 2, 3), float(s)) for s in mine])
        g = gather_results(poses, verts, Sn * world, "block")
        gathered = None if g is None else int(g[0].shape[0])
        ok = None if g is None else bool(all((g[0][s] == s).all() for s in range(Sn * world)))
    else:
        gathered, ok = None, None
    if rank == 0:
        print(json.dumps({"metric": METRIC, "dry_run": True, "value": None, "unit": "frames/s", "n_gpus": world,
                          "steps": K, "ms_per_step": ms / max(K, 1), "config": workload(args, world),
                          "shards": [assign_streams(Sn * world, world, r, "block") for r in range(world)],
                          "gathered_streams": gathered, "gather_ok": ok}))
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    if args.dry_run:
        run_dry(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
