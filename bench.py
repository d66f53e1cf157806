#!/usr/bin/env python
"""Benchmark: boxes ranged/s & stereo frames/s at 1920x1080 with 64 boxes
(BASELINE.json metric, config C2), p50 frame latency, on N GPUs.

One step = the hot path (census -> planner -> fused sampler/matcher with
forward-backward verification and sub-pixel fit -> aggregation + range) over
a batch of F synthetic C2 frames resident in HBM, followed by the NCCL gather
of the per-box results to rank 0 (frames shard across ranks: weak scaling).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--frames F]
  python bench.py --impl reference      # the reference's CPU path on the host cores

Prints one JSON line (rank 0).  Needs the CUDA library (build() first).
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

METRIC = "boxes ranged/sec & stereo frames/sec at 1920x1080, 64 boxes; p50 frame latency"
W, H = 1920, 1080
CENSUS_BYTES_PER_FRAME = 2 * (W * H + 4 * W * H + 4 * (W // 2) * (H // 2))  # 24,883,200
POPC_PER_CLK_PER_SM = 16  # CUDA programming guide throughput table (cc 8.x-9.0)


def popc_peak_per_clk():
    """Measured XOR+POPC+IADD evaluations per clock per SM on this GPU model
    (tools/popc_probe.cu -> profiles/r1_popc_probe.json), else the nominal 16."""
    try:
        with open(os.path.join(ROOT, "profiles", "r1_popc_probe.json")) as f:
            return float(json.load(f)["evals_per_clk_per_sm"]), "measured (tools/popc_probe.cu)"
    except Exception:
        return float(POPC_PER_CLK_PER_SM), "nominal"
N_SM = 148


def census_required_bytes(dets, w, h, tau_s=48.0, scale=2, dx_far=256, dx_close=256, code_bytes=4, rx=2, ry=2):
    """Bytes K1 must move for one frame.  The reference's ROI census
    (census_transform_rois, template_match.hpp:245-321) computes full codes
    inside the FAR ROI rectangles (box dilated by dx_max_far + 2 columns and 3
    rows) and reduced codes inside the CLOSE ROI rectangles (reduced
    coordinates, dilated by ceil(dx_max_close / s) + 2 and 3) of both images.
    K1 computes the part of each rectangle the matcher can read
    (read_rect, census.cu): on the left image the box rows across
    [x0 - dx_max, x1 + dx_max], on the right image the box rows +-1 across
    [x0 - dx_max, x1].  Algorithmic bytes = code_bytes
    per such code (4; 8 for the 9x7 extension) + every image byte under those
    codes' (2 rx + 1) x (2 ry + 1) windows (source pixels for the reduced
    raster), read once.  -> dict."""
    import math
    cw, ch = w // scale, h // scale
    sx, sy = cw / w, ch / h
    dxs = (dx_close + scale - 1) // scale
    ref_f, ref_r = np.zeros((h, w), bool), np.zeros((ch, cw), bool)
    need = [[np.zeros((h, w), bool), np.zeros((ch, cw), bool)] for _ in range(2)]  # [image][raster]
    for d in dets:
        x0, x1 = (d.cx - d.w / 2) * w, (d.cx + d.w / 2) * w
        y0, y1 = (d.cy - d.h / 2) * h, (d.cy + d.h / 2) * h
        if max(d.w * w, d.h * h) < tau_s:  # classify_far_close
            k, W, H, dxm, ref = 0, w, h, dx_far + 2, ref_f
            bx0, bx1, by0, by1 = math.floor(x0), math.ceil(x1), math.floor(y0), math.ceil(y1)
        else:
            k, W, H, dxm, ref = 1, cw, ch, dxs + 2, ref_r
            bx0, bx1 = math.floor(x0 * sx), math.ceil(x1 * sx)
            by0, by1 = math.floor(y0 * sy), math.ceil(y1 * sy)
        a, e = max(0, by0 - 3), min(H, by1 + 4)
        c0, c1 = max(0, bx0 - dxm), min(W, bx1 + dxm + 1)
        ref[a:e, c0:c1] = True
        dxr = dxm - 2  # census.cu read_rect (tight 2)
        need[0][k][max(a, by0):min(e, by1 + 1), max(c0, bx0 - dxr):min(c1, bx1 + dxr + 1)] = True
        need[1][k][max(a, by0 - 1):min(e, by1 + 2), max(c0, bx0 - dxr):min(c1, bx1 + 1)] = True
    codes, reads = 0, 0
    for img in range(2):
        nf, nr = need[img]
        codes += int(nf.sum()) + int(nr.sum())
        # image pixels under the windows: the code masks (reduced code
        # (x', y') at source (2x', 2y')) dilated by ry rows / rx columns
        m = nf.copy()
        m[:scale * ch:scale, :scale * cw:scale] |= nr
        for ax, r in ((0, ry), (1, rx)):
            p = np.pad(m, [(r, r) if a == ax else (0, 0) for a in (0, 1)])
            n = m.shape[ax]
            m = np.zeros_like(m)
            for o in range(2 * r + 1):
                m |= p[o:o + n, :] if ax == 0 else p[:, o:o + n]
        reads += int(m.sum())
    return {"bytes": code_bytes * codes + reads, "codes": codes, "image_bytes": reads,
            "ref_full_codes": int(ref_f.sum()), "ref_reduced_codes": int(ref_r.sum()),
            "ref_bytes": 2 * (w * h + code_bytes * int(ref_f.sum()) + code_bytes * int(ref_r.sum()))}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), float(p.get("sm_max_mhz", 1965.0)), "measured"
    except Exception:
        return 6650.0, 1965.0, "fallback"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region: NVML
    (nvidia_ml_py) polled every 5 ms from a thread, or nvidia-smi -lms as a
    fallback.  start() returns once the first sample is in."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,utilization.gpu")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
    BITS = [0x8, 0x40, 0x20, 0x4]  # nvmlClocksEventReason*

    def __init__(self, index: int):
        self.index, self.rows, self.proc, self.nvml = index, [], None, None
        self.stop_ev = threading.Event()

    def _nvml_handle(self):
        import pynvml
        pynvml.nvmlInit()
        try:  # the CUDA device's UUID (CUDA_VISIBLE_DEVICES may renumber)
            import torch
            uuid = str(torch.cuda.get_device_properties(self.index).uuid)
            return pynvml, pynvml.nvmlDeviceGetHandleByUUID("GPU-" + uuid)
        except Exception:
            return pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.index)

    def _poll(self):
        nv, h = self.nvml
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        while not self.stop_ev.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                ut = nv.nvmlDeviceGetUtilizationRates(h).gpu
                self.rows.append([str(sm), str(mx)] + ["Active" if rs & b else "Not Active" for b in self.BITS]
                                 + [str(ut)])
            except Exception:
                pass
            self.stop_ev.wait(0.005)

    def start(self):
        try:
            self.nvml = self._nvml_handle()
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
        except Exception:
            self.nvml = None
            try:
                self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                              "--format=csv,noheader,nounits", "-lms", "50"],
                                             stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
                self.t = threading.Thread(target=self._read, daemon=True)
                self.t.start()
            except Exception:
                self.proc = None
        t0 = time.time()
        while not self.rows and time.time() - t0 < 15 and (self.nvml or self.proc):
            time.sleep(0.01)
        self.skip = len(self.rows)  # samples taken before the timed region

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def stop(self):
        self.stop_ev.set()
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.nvml:
            self.t.join(timeout=1)
        rows = self.rows[self.skip:] or self.rows[-1:]
        busy = [r for r in rows if r[6].isdigit() and int(r[6]) > 0] or rows
        sm = [float(r[0]) for r in busy if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        reasons = sorted({self.NAMES[i] for r in rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows), "source": "nvml" if self.nvml else "nvidia-smi"}


# ------------------------------------------------------------------ shared
def workload_config(F: int, world: int) -> dict:
    """The `config` both arms print (same_config): the C2 workload, frames per
    step per GPU and how the frames are seeded."""
    return {"workload": "C2: 1920x1080 rendered stereo pairs (render_stereo_pair), 64 boxes (48 FAR + 16 CLOSE), "
                        "dx_max_far = dx_max_close = 256, tau_v 1.0, fwd-bwd + sub-pixel, range z",
            "frames_per_step_per_gpu": F, "noise_sigma": 2.0,
            "frame_seeds": "global frame g = rank * frames_per_step + i has seed 1 + g (all distinct)",
            "l2": f"inputs {2 * F * W * H / 1e6:.0f} MB per step per GPU (every frame distinct) > 126 MB L2 "
                  f"(no flush needed)",
            "parallelism": f"frame-sharded dp{world}, per-box results all_gathered"}


def ref_arm():
    """oracle/ref_arm.py: the reference compiled in place, no product import."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import ref_arm as ra
    return ra


def free_port() -> int:
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def spawn_ranks(n: int) -> int:
    """--gpus N without WORLD_SIZE: re-exec this command under
    torch.distributed.run with N ranks (one per GPU) on 127.0.0.1."""
    import torch
    have = torch.cuda.device_count()
    if n > have:
        print(json.dumps({"metric": METRIC, "error": f"--gpus {n} but only {have} CUDA device(s) visible"}))
        return 1
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def compare_records(got_recs, got_cnt, want_recs, want_cnt):
    """Per-frame bytewise comparison of rg_object_disparity rows -> (frame
    mismatches, box mismatches)."""
    bad_f = bad_b = 0
    for f in range(len(want_cnt)):
        n = int(want_cnt[f])
        if int(got_cnt[f]) != n:
            bad_f += 1
            bad_b += max(n, int(got_cnt[f]))
            continue
        g = np.frombuffer(bytes(got_recs[f][:32 * n]), np.uint8).reshape(n, 32)
        w = np.frombuffer(want_recs[f][:n].tobytes(), np.uint8).reshape(n, 32)
        d = int((g != w).any(axis=1).sum())
        bad_b += d
        bad_f += int(d > 0)
    return bad_f, bad_b


# ------------------------------------------------------------------ C5 stream
def c5_stream(args, eng, ctx, dev, stream, rank, world, dets, recs_np, offs_np):
    """BASELINE config 4 (C5): a stream of N distinct C2 frames (seeds 1..N)
    sharded contiguously over the ranks, each shard rendered in HBM by the
    device frame source (untimed), ranged in chunks of --frames and the
    per-box results all_gathered -- shard.run_stream / gather_slabs /
    frame_order / gathered_boxes, the functions tests/test_dist_cpu.py runs at
    world 2.  Strong scaling.  Timed with CUDA events, max over ranks.  Then
    every (N/256)-th frame is re-ranged by the reference on the host cores
    and compared with the gathered records."""
    import torch
    import torch.distributed as dist
    from paper_2604_07980_b200 import shard, synth as S
    from paper_2604_07980_b200.engine import OUT_DTYPE

    N, chunk = args.stream_frames, args.frames
    lo, hi = shard.shard_bounds(N, rank, world)
    n = hi - lo
    rec = eng.out_stride * OUT_DTYPE.itemsize
    dL = torch.empty((max(n, 1), H, W), dtype=torch.uint8, device=dev)
    dR = torch.empty_like(dL)
    r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    r0.record(stream)
    for c0 in range(0, n, 512):
        c1 = min(n, c0 + 512)
        S.render_frames_device(ctx, [S.scene_c2(seed=1 + f, noise=2.0)[0] for f in range(lo + c0, lo + c1)],
                               dL[c0:], dR[c0:], stream=stream.cuda_stream)
    r1.record(stream)
    d_dets = torch.from_numpy(np.tile(recs_np[offs_np[0]:offs_np[1]], chunk).view(np.uint8)).to(dev)
    d_offs = torch.from_numpy((np.arange(chunk + 1) * len(dets)).astype(np.int32)).to(dev)
    out, cnt, g_out, g_cnt = shard.alloc_slabs(N, world, rec, device=dev)

    def range_chunk(glo, ghi, o, c):
        a = glo - lo
        eng.range_device(dL[a:a + ghi - glo], dR[a:a + ghi - glo], d_dets, d_offs[:ghi - glo + 1], o, c,
                         stream=stream.cuda_stream, sync=False)

    def run():
        shard.run_stream(range_chunk, N, rank, world, chunk, out, cnt, rec)
        shard.gather_slabs(out, cnt, g_out, g_cnt, world)
        assert ctx.sync() == 0, "C5: a batch overflowed the block list"

    run()  # warm-up pass (allocations for the tail chunk)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    run()
    e1.record(stream)
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1), r0.elapsed_time(r1)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms, render_ms = float(t[0]), float(t[1])
    boxes = shard.gathered_boxes(g_cnt, N, world)
    # parity sample: every (N/256)-th global frame, checked by its owner rank
    parity = {"checked_frames": 0, "frame_mismatches": 0, "box_mismatches": 0}
    if not args.no_parity:
        ra = ref_arm()
        step_s = max(1, N // args.parity_c5_frames)
        mine = [g for g in range(0, N, step_s) if lo <= g < hi]
        recs_all, cnt_all = shard.frame_order(g_out, g_cnt, N, world, rec)
        if mine and ra.have_reference():
            idx = torch.tensor([g - lo for g in mine], device=dev)
            hL, hR = dL[idx].cpu().numpy(), dR[idx].cpu().numpy()
            pr, po = np.tile(recs_np[offs_np[0]:offs_np[1]], len(mine)), \
                (np.arange(len(mine) + 1) * len(dets)).astype(np.int32)
            _, want, wcnt = ra.range_frames(hL, hR, pr, po, ra.ranger_config_c2(), ra.cpu_threads(), eng.out_stride)
            bf, bb = compare_records(recs_all[mine], cnt_all[mine], want, wcnt)
            parity = {"checked_frames": len(mine), "frame_mismatches": bf, "box_mismatches": bb}
        pt = torch.tensor([parity["checked_frames"], parity["frame_mismatches"], parity["box_mismatches"]],
                          dtype=torch.int64, device=dev)
        if world > 1:
            dist.all_reduce(pt)
        parity = {"checked_frames": int(pt[0]), "frame_mismatches": int(pt[1]), "box_mismatches": int(pt[2]),
                  "sample": f"every {step_s}-th frame of the stream, re-ranged by oracle/_ref (the reference "
                            "compiled in place) on the owner rank's host cores, vs the gathered records",
                  "checker": "reference" if ra.have_reference() else "unavailable"}
    del dL, dR
    return {"config": f"C5: {N} distinct C2 frames (device-rendered, seeds 1..{N}, noise 2.0) sharded contiguously "
                      f"over {world} rank(s), ranged in chunks of {chunk}, per-box results all_gathered",
            "frames": N, "ms": ms, "frames_per_sec": N / (ms / 1e3), "boxes": boxes,
            "boxes_per_sec": boxes / (ms / 1e3), "scaling": "strong", "render_ms_per_rank": render_ms,
            "parity": parity}


# ------------------------------------------------------------------ other BASELINE configs
def config_c3(args, ctx, dev, stream):
    """C3 (BASELINE config 2): 2880x1860, 256 boxes (192 FAR in 96 occluded
    pairs + 64 CLOSE), occlusion-aware sampling, CLOSE median aggregation;
    device-rendered distinct frames, one rg_range_frames per step; the first
    frames re-ranged by the reference for parity."""
    import torch
    from paper_2604_07980_b200 import synth as S
    from paper_2604_07980_b200.engine import OUT_DTYPE, FrameEngine, pack_detections

    F3 = args.c3_frames
    sc0, cfg = S.scene_c3(seed=1, noise=2.0)
    w, h = sc0.width, sc0.height
    scenes = [S.scene_c3(seed=1 + i, noise=2.0)[0] for i in range(F3)]
    dets = S.ground_truth_detections(scenes[0])
    dL = torch.empty((F3, h, w), dtype=torch.uint8, device=dev)
    dR = torch.empty_like(dL)
    S.render_frames_device(ctx, scenes, dL, dR, stream=stream.cuda_stream)
    eng = FrameEngine(w, h, cfg, len(dets), S.F_PX, S.BASELINE_M, ctx=ctx)
    recs, offs = pack_detections([dets] * F3)
    d_dets = torch.from_numpy(recs.view(np.uint8)).to(dev)
    d_offs = torch.from_numpy(offs).to(dev)
    out = torch.zeros(F3 * eng.out_stride * OUT_DTYPE.itemsize, dtype=torch.uint8, device=dev)
    cnt = torch.zeros(F3, dtype=torch.int32, device=dev)
    step = lambda: eng.range_device(dL, dR, d_dets, d_offs, out, cnt, stream=stream.cuda_stream,  # noqa: E731
                                    sync=False)
    for _ in range(3):
        step()
        ctx.sync()
    step()
    assert ctx.sync() == 0
    torch.cuda.synchronize()
    ctx.reset_counters()
    reps = max(3, min(args.steps, 10))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        step()
    e1.record(stream)
    assert ctx.sync() == 0
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    evals, _ = ctx.work()
    boxes = int(cnt.sum().item())
    res = {"config": f"C3: {w}x{h}, {len(dets)} boxes (192 FAR incl. 96 occluded + 64 CLOSE), dx_max 256, "
                     f"{F3} device-rendered distinct frames (noise 2.0) per rg_range_frames call",
           "ms_per_step": ms, "boxes_per_sec": boxes / (ms / 1e3), "frames_per_sec": F3 / (ms / 1e3),
           "valid_boxes_per_frame": None, "hamming_evals_per_frame": evals / (reps * F3)}
    o = np.frombuffer(out.cpu().numpy().tobytes(), OUT_DTYPE).reshape(F3, eng.out_stride)
    c = cnt.cpu().numpy()
    res["valid_boxes_per_frame"] = float(np.mean([o[f, :c[f]]["valid"].sum() for f in range(F3)]))
    if not args.no_parity:
        ra = ref_arm()
        if ra.have_reference():
            k = min(F3, args.c3_parity_frames)
            hL, hR = dL[:k].cpu().numpy(), dR[:k].cpu().numpy()
            _, want, wcnt = ra.range_frames(hL, hR, recs[:offs[k]], offs[:k + 1], cfg.to_c(), ra.cpu_threads(),
                                            eng.out_stride)
            got = out.cpu().numpy().reshape(F3, -1)
            bf, bb = compare_records(got[:k], c[:k], want, wcnt)
            res["parity"] = {"checked_frames": k, "frame_mismatches": bf, "box_mismatches": bb,
                             "checker": "reference (oracle/_ref)"}
    del dL, dR
    return res


def config_c1_9x7(args, ctx, dev, stream):
    """C1 (BASELINE config 0) with the 9x7 / uint64 census extension: 640x480,
    8 boxes at integer disparities, dx_max 64; parity against the C
    restatement (the reference has no 9x7 window: parity unpinned)."""
    import torch
    from paper_2604_07980_b200 import _abi, synth as S
    from paper_2604_07980_b200.engine import OUT_DTYPE, FrameEngine, pack_detections

    F1 = args.c1_frames
    sc0, cfg = S.scene_c1(seed=1, noise=2.0)
    cfg.census_9x7 = True
    w, h = sc0.width, sc0.height
    scenes = [S.scene_c1(seed=1 + i, noise=2.0)[0] for i in range(F1)]
    dets = S.ground_truth_detections(scenes[0])
    dL = torch.empty((F1, h, w), dtype=torch.uint8, device=dev)
    dR = torch.empty_like(dL)
    S.render_frames_device(ctx, scenes, dL, dR, stream=stream.cuda_stream)
    eng = FrameEngine(w, h, cfg, len(dets), S.F_PX, S.BASELINE_M, ctx=ctx)
    recs, offs = pack_detections([dets] * F1)
    d_dets = torch.from_numpy(recs.view(np.uint8)).to(dev)
    d_offs = torch.from_numpy(offs).to(dev)
    out = torch.zeros(F1 * eng.out_stride * OUT_DTYPE.itemsize, dtype=torch.uint8, device=dev)
    cnt = torch.zeros(F1, dtype=torch.int32, device=dev)
    step = lambda: eng.range_device(dL, dR, d_dets, d_offs, out, cnt, stream=stream.cuda_stream)  # noqa: E731
    for _ in range(3):
        step()  # sync=True: resubmits a batch that overflowed
    torch.cuda.synchronize()
    ctx.reset_counters()
    ctx.set_profiling(True)  # profiling: every batch blocks
    reps = max(3, min(args.steps, 10))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    ctx.set_profiling(False)
    stage_ms, stage_launches, _ = ctx.counters()
    ms = e0.elapsed_time(e1) / reps
    boxes = int(cnt.sum().item())
    full_bytes = 2 * (w * h + 8 * w * h + 8 * (w // 2) * (h // 2))  # B = 8 for 9x7
    req = census_required_bytes(dets, w, h, cfg.tau_s, cfg.close_scale, cfg.dx_max_far, cfg.dx_max_close,
                                code_bytes=8, rx=4, ry=3)
    cen_ms = stage_ms[0] / reps  # per call (the ROI census is 3 kernel launches)
    res = {"config": f"C1 9x7: {w}x{h}, {len(dets)} boxes (5 FAR + 3 CLOSE) at integer disparities, dx_max 64, "
                     f"9x7 census / uint64 descriptors, {F1} device-rendered distinct frames (noise 2.0) per call",
           "ms_per_step": ms, "boxes_per_sec": boxes / (ms / 1e3), "frames_per_sec": F1 / (ms / 1e3),
           "census64": {"ms_per_launch": cen_ms, "kernel": "census_rows_kernel + census64_rowtile_kernel<1, 2> "
                                                           "(ROI tiles of the matcher's read sets)",
                        "achieved_gbs": req["bytes"] * F1 / (cen_ms / 1e3) / 1e9,
                        "algorithmic_bytes_per_frame": req["bytes"],
                        "algorithmic_bytes": f"{req['codes']} 8-B codes per frame (both images) + the "
                                             f"{req['image_bytes']} image bytes under their 9x7 windows",
                        "full_frame_equivalent_gbs": full_bytes * F1 / (cen_ms / 1e3) / 1e9}}
    if not args.no_parity:
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        import oracle_lib
        k = min(F1, 8)
        hL, hR = dL[:k].cpu().numpy(), dR[:k].cpu().numpy()
        got = out.cpu().numpy().reshape(F1, -1)
        c = cnt.cpu().numpy()
        bad_f = 0
        for f in range(k):
            want, _ = oracle_lib.oracle().estimate(hL[f], hR[f], [_abi.Detection(d.cx, d.cy, d.w, d.h, d.class_id,
                                                                                 d.id) for d in dets],
                                                   cfg.to_c(), S.F_PX, S.BASELINE_M)
            wb = b"".join(bytes(x) for x in want)
            bad_f += int(int(c[f]) != len(want) or bytes(got[f][:len(wb)]) != wb)
        res["parity"] = {"checked_frames": k, "frame_mismatches": bad_f,
                         "checker": "oracle restatement (9x7 parity unpinned: no reference 9x7 window)"}
    del dL, dR
    return res


# ------------------------------------------------------------------ reference arm
def run_reference(args):
    """Reference arm: the reference's own render_stereo_pair and
    estimate_object_disparities (compiled in place into oracle/_ref; no
    product library loaded), all host threads, frame-parallel (one whole frame
    per thread at workers = 1), on the GPU arm's rank-0 step: the same
    --frames C2 frames (seeds 1..F), K timed steps after W warm-up steps."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    if rank != 0:
        return 0
    ra = ref_arm()
    if not ra.have_reference():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libranger_ref.so not built"}))
        return 0
    threads = ra.cpu_threads()
    F = args.frames
    L, R, dets, offs = ra.render([ra.scene_c2(1 + i, 2.0) for i in range(F)], threads)
    cfg = ra.ranger_config_c2()
    out_stride = 64
    secs, boxes = [], 0
    for i in range(args.warmup + args.steps):
        t, _, cnt = ra.range_frames(L, R, dets, offs, cfg, threads, out_stride)
        if i >= args.warmup:
            secs.append(t)
            boxes += int(cnt.sum())
    total = sum(secs)
    val = boxes / total
    sample = (f"{F} C2 frames per step (seeds 1..{F}, noise 2.0) rendered by the reference's render_stereo_pair, "
              f"ranged one per host thread at workers=1 (frame-parallel) by the reference's "
              f"estimate_object_disparities from oracle/_ref, {len(secs)} steps, {total:.1f} s")
    line = {
        "metric": METRIC, "impl": "reference", "value": val, "unit": "boxes/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * total / len(secs),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8/u32/f64",
        "data": "synthetic", "frames_per_sec": F * len(secs) / total,
        "config": workload_config(F, world),
        "cpu_baseline": {"value": val, "unit": "boxes/s", "cores": threads, "kind": "reference", "sample": sample,
                         "cpu_model": ra.cpu_model()},
        "e2e": {"value": val, "unit": "boxes/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


def cpu_reference_run(L, R, dets_np, offs_np, seconds: float):
    """cpu_baseline: the reference (oracle/_ref) on the host cores,
    frame-parallel (SURVEY 8(d) mode iii), bounded in time, plus the
    reference's per-stage times on one frame at workers = 1 and = nproc."""
    import ctypes as C
    ra = ref_arm()
    if not ra.have_reference():
        return None
    threads = ra.cpu_threads()
    cfg = ra.ranger_config_c2()
    n = L.shape[0]
    frames, wall, boxes = 0, 0.0, 0
    while wall < seconds:
        t, _, cnt = ra.range_frames(L, R, dets_np, offs_np, cfg, threads, 64)
        wall += t
        frames += n
        boxes += int(cnt.sum())
    res = {"value": boxes / wall, "unit": "boxes/s", "frames_per_sec": frames / wall, "cores": threads,
           "cpu_model": ra.cpu_model(), "kind": "reference",
           "sample": f"{frames} C2 frames ({n} distinct, noise 2.0) ranged by the reference's "
                     f"estimate_object_disparities, {threads} threads x whole frames at workers=1, {wall:.1f} s"}
    try:
        lib = ra.lib()
        d0 = np.ascontiguousarray(dets_np[offs_np[0]:offs_np[1]])

        class Rect(C.Structure):
            _fields_ = [("x0", C.c_int32), ("y0", C.c_int32), ("x1", C.c_int32), ("y1", C.c_int32)]

        class Bm(C.Structure):
            _fields_ = [("num_disparities", C.c_int32), ("block_size", C.c_int32), ("min_disparity", C.c_int32),
                        ("downscale", C.c_int32), ("texture_threshold", C.c_double),
                        ("uniqueness_ratio", C.c_double)]
        roi, bm = Rect(480, 270, 1440, 810), Bm(32, 9, -4, 1, 10.0, 10.0)
        detail = {}
        lib.ref_bench_stages.restype = C.c_int
        for wk, reps, rr in ((1, 3, 1), (threads, 5, 2)):
            t = (C.c_double * 3)()
            st = lib.ref_bench_stages(C.c_void_p(L[0].ctypes.data), C.c_void_p(R[0].ctypes.data), W, H,
                                      C.c_void_p(d0.ctypes.data), len(d0), C.byref(cfg), wk, reps, C.byref(roi),
                                      -8, 8, C.byref(bm), rr, t)
            if st == 0:
                detail[f"workers_{wk}"] = {"estimate_ms_per_frame": 1e3 * t[0], "census_x2_ms": 1e3 * t[1],
                                           "autorect_c4_ms": 1e3 * t[2]}
        res["stages_one_frame"] = detail
    except Exception as e:  # pragma: no cover
        res["stages_one_frame"] = f"error: {e}"
    return res


# ------------------------------------------------------------------ our arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--frames", type=int, default=256, help="frames per step per GPU")
    ap.add_argument("--stream-frames", type=int, default=4096,
                    help="C5: frames in the sharded stream measurement (0: skip)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-parity", action="store_true", help="skip the parity sweeps against oracle/_ref")
    ap.add_argument("--parity-c5-frames", type=int, default=256)
    ap.add_argument("--latency-runs", type=int, default=1000)
    ap.add_argument("--e2e-chunk", type=int, default=64, help="frames per rg_range_frames_host chunk")
    ap.add_argument("--c3-frames", type=int, default=32, help="C3 frames per call (0: skip the C3 line)")
    ap.add_argument("--c3-parity-frames", type=int, default=16)
    ap.add_argument("--c1-frames", type=int, default=1024, help="9x7 C1 frames per call (0: skip)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args.gpus)

    import torch
    import torch.distributed as dist

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    assert world == args.gpus, f"WORLD_SIZE {world} != --gpus {args.gpus}"
    assert world <= torch.cuda.device_count(), f"{world} ranks but {torch.cuda.device_count()} CUDA devices"
    torch.cuda.set_device(local)
    os.environ["RG_DEVICE"] = str(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_2604_07980_b200 import ranger as rg, shard
    from paper_2604_07980_b200.engine import OUT_DTYPE, FrameEngine, pack_detections
    from paper_2604_07980_b200 import synth as S

    F = args.frames
    ctx = rg.Context(local)
    dev = torch.device("cuda", local)
    # the ring is this rank's shard of a (world x F)-frame stream: global frame
    # g = rank * F + i, seed 1 + g, every frame distinct, rendered in HBM by the
    # device frame source (byte-identical to the reference renderer,
    # tests/test_gpu_render.py, tests/test_ref_arm.py)
    lo, hi = shard.shard_bounds(F * world, rank, world)
    scenes = [S.scene_c2(seed=1 + g, noise=2.0)[0] for g in range(lo, hi)]
    dets, cfg = S.ground_truth_detections(scenes[0]), S.scene_c2(seed=1)[1]
    dL = torch.empty((F, H, W), dtype=torch.uint8, device=dev)
    dR = torch.empty_like(dL)
    S.render_frames_device(ctx, scenes, dL, dR)
    torch.cuda.synchronize()
    L, R = dL.cpu().numpy(), dR.cpu().numpy()  # host copies: e2e feed, CPU baseline, parity sweep
    n_boxes = len(dets)
    eng = FrameEngine(W, H, cfg, n_boxes, S.F_PX, S.BASELINE_M, ctx=ctx)
    rec = eng.out_stride * OUT_DTYPE.itemsize
    recs, offs = pack_detections([dets] * F)
    d_dets = torch.from_numpy(recs.view(np.uint8)).to(dev)
    d_offs = torch.from_numpy(offs).to(dev)
    d_out, d_cnt, g_out, g_cnt = shard.alloc_slabs(F * world, world, rec, device=dev)
    # a real (non-legacy-default) stream: the library launches on it and the
    # CUDA events below are recorded on it
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)

    def range_chunk(glo, ghi, o, c):  # asynchronous; ctx.sync() after the timed loop
        eng.range_device(dL, dR, d_dets, d_offs, o, c, stream=stream.cuda_stream, sync=False)

    def step():  # the shard's F frames, then the per-box results to every rank
        shard.run_stream(range_chunk, F * world, rank, world, F, d_out, d_cnt, rec)
        shard.gather_slabs(d_out, d_cnt, g_out, g_cnt, world)

    # ---- warmup (a first batch that overflows grows the device block list)
    for _ in range(args.warmup):
        step()
        ctx.sync()
    step()
    assert ctx.sync() == 0, "the block list still overflows after the warm-up"
    torch.cuda.synchronize()

    # ---- timed region (device-resident feed, default one-stream schedule)
    ctx.reset_counters()
    clocks = ClockSampler(local)
    clocks.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    overflow_in_timed = ctx.sync()  # 0: every timed batch produced its results
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    clk = clocks.stop()
    _, _, total_launches = ctx.counters()
    evals, blocks = ctx.work()
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    boxes_step = shard.gathered_boxes(g_cnt, F * world, world)
    value = boxes_step * args.steps / (ms_max / 1000.0)
    fps = F * args.steps * world / (ms_max / 1000.0)

    # ---- kernel rooflines: the same steps with per-stage CUDA events, each
    # step read out alone; stage times are the per-stage medians over the
    # steps (robust to a one-off disturbance of a single step)
    roof_steps = max(3, min(args.steps, 10))
    per_step, r_evals = [], 0
    ctx.set_profiling(True)
    for _ in range(roof_steps):
        ctx.reset_counters()
        step()
        torch.cuda.synchronize()
        per_step.append(ctx.counters()[0])
        r_evals += ctx.work()[0]
    ctx.set_profiling(False)
    stage_ms = [statistics.median(p[i] for p in per_step) * roof_steps for i in range(len(per_step[0]))]
    # the full-frame census kernel (census_pairs_kernel: batches under 12
    # frames, the single-image API, SGM) on the same 256-frame steps
    # (rg_set_census_rois(0)): SURVEY 8(d)'s full-frame bytes over its time
    ctx.set_census_rois(False)
    step()
    assert ctx.sync() == 0
    torch.cuda.synchronize()
    ctx.reset_counters()
    ctx.set_profiling(True)
    for _ in range(roof_steps):
        step()
    torch.cuda.synchronize()
    ctx.set_profiling(False)
    ctx.set_census_rois(True)
    ff = F
    ff_ms = ctx.counters()[0][0] / roof_steps

    # ---- parity sweep: every ring frame of every rank, re-ranged by the
    # reference (oracle/_ref) on the host cores, vs the gathered records
    parity = None
    if not args.no_parity:
        ra = ref_arm()
        bf = bb = 0
        if ra.have_reference():
            recs_all, cnt_all = shard.frame_order(g_out, g_cnt, F * world, world, rec)
            _, want, wcnt = ra.range_frames(L, R, recs, offs, cfg.to_c(), ra.cpu_threads(), eng.out_stride)
            bf, bb = compare_records(recs_all[lo:hi], cnt_all[lo:hi], want, wcnt)
        pt = torch.tensor([hi - lo if ra.have_reference() else 0, bf, bb], dtype=torch.int64, device=dev)
        if world > 1:
            dist.all_reduce(pt)
        parity = {"checked_frames": int(pt[0]), "frame_mismatches": int(pt[1]), "box_mismatches": int(pt[2]),
                  "sample": "every ring frame of every rank (the timed step's output, after the gather)",
                  "checker": "reference (oracle/_ref, compiled in place)" if ra.have_reference() else "unavailable"}

    # ---- end-to-end through the public host API (pinned host frames, H2D/D2H inside)
    keep = []

    def pin(a):  # pinned host copy of any numpy array (structured dtypes included)
        t = torch.empty(a.nbytes, dtype=torch.uint8).pin_memory()
        keep.append(t)
        v = t.numpy().view(a.dtype).reshape(a.shape)
        v[...] = a
        return v
    hL, hR = pin(L), pin(R)
    h_recs, h_offs = pin(recs), pin(offs)
    h_out = pin(np.zeros(F * eng.out_stride, OUT_DTYPE))
    h_cnt = pin(np.zeros(F, np.int32))
    for _ in range(2):
        eng.range_host(hL, hR, h_recs, h_offs, h_out, h_cnt, chunk=args.e2e_chunk, stream=stream.cuda_stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    x0 = ctx.transfer()
    t0 = time.perf_counter()
    e2e_steps = max(2, args.steps // 2)
    for _ in range(e2e_steps):
        eng.range_host(hL, hR, h_recs, h_offs, h_out, h_cnt, chunk=args.e2e_chunk, stream=stream.cuda_stream)
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    x1 = ctx.transfer()
    te = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = int(h_cnt.sum()) * e2e_steps * world / float(te.item())
    e2e_parity = bool(h_out.tobytes() == d_out.cpu().numpy().tobytes()[:h_out.nbytes])
    # bytes the library moved per step (rg_get_transfer): the zero-copy
    # gathers fetch only the image bytes the ROI census reads
    h2d = (x1[0] - x0[0]) // e2e_steps
    d2h = (x1[1] - x0[1]) // e2e_steps
    h2d_full = int(hL.nbytes + hR.nbytes + h_recs.nbytes + h_offs.nbytes)
    # the e2e bound: this box's pinned host -> device copy bandwidth (one
    # 256 MiB copy stream, CUDA events, best of 6 x 16 copies)
    pcie_gbs = None
    try:
        ph = torch.empty(256 << 20, dtype=torch.uint8).pin_memory()
        pd = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
        best = 0.0
        for _ in range(6):
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record(stream)
            with torch.cuda.stream(stream):
                for _ in range(16):
                    pd.copy_(ph, non_blocking=True)
            a1.record(stream)
            torch.cuda.synchronize()
            best = max(best, 16 * ph.nbytes / (a0.elapsed_time(a1) * 1e-3) / 1e9)
        pcie_gbs = best
        del ph, pd
    except Exception:  # pragma: no cover
        pass
    e2e_h2d_gbs = h2d * e2e_steps / float(te.item()) / 1e9

    # ---- p50 latency: one frame, host in -> per-box results on host
    lat = []
    for i in range(args.latency_runs):
        a = time.perf_counter()
        eng.range_host(hL[i % F:i % F + 1], hR[i % F:i % F + 1], h_recs[:n_boxes], h_offs[:2], h_out[:eng.out_stride],
                       h_cnt[:1], chunk=1, stream=stream.cuda_stream)
        lat.append(time.perf_counter() - a)
    lat_dev = []
    for i in range(args.latency_runs):
        a = time.perf_counter()
        eng.range_device(dL[i % F:i % F + 1], dR[i % F:i % F + 1], d_dets, d_offs[:2], d_out, d_cnt,
                         stream=stream.cuda_stream)
        torch.cuda.synchronize()
        lat_dev.append(time.perf_counter() - a)

    # ---- auto-rectification offset search (config C4), timed separately
    rect = None
    try:
        nrf = 8
        best = torch.zeros(nrf, dtype=torch.int32, device=dev)
        cnts = torch.zeros(nrf * 17, dtype=torch.int64, device=dev)
        for _ in range(2):
            eng.auto_rect_device(dL[:nrf], dR[:nrf], S.C4_ROI, -8, 8, S.c4_bm(), best, cnts, stream=stream.cuda_stream)
        torch.cuda.synchronize()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        reps = 3
        for _ in range(reps):
            eng.auto_rect_device(dL[:nrf], dR[:nrf], S.C4_ROI, -8, 8, S.c4_bm(), best, cnts, stream=stream.cuda_stream)
        a1.record(stream)
        torch.cuda.synchronize()
        rms = a0.elapsed_time(a1) / (reps * nrf)
        cells = 960 * 540 * 32 * 17
        rect = {"config": "C4: 960x540 ROI, 32 disparities (d_min -4), 9x9 SAD, delta -8..8",
                "ms_per_frame": rms, "frames_per_sec": 1000.0 / rms,
                "window_evals_per_sec": cells / (rms / 1000.0), "delta_star_frame0": int(best[0].item())}
    except Exception as e:  # pragma: no cover
        rect = {"error": str(e)}

    # ---- the full TEMPLATE_MATCHER frame loop (rg_range_sequence): offset
    # search on every uncorrected pair (RectSearchConfig defaults: delta -3..3,
    # central half, 32 disparities) + filter scan + corrected ranging
    seq = None
    try:
        nsf = min(F, 64)
        rect_cfg = rg.RectSearchConfig()
        seq_out = torch.zeros(nsf * eng.out_stride * OUT_DTYPE.itemsize, dtype=torch.uint8, device=dev)
        seq_cnt = torch.zeros(nsf, dtype=torch.int32, device=dev)
        seq_offs = torch.from_numpy(pack_detections([dets] * nsf)[1]).to(dev)
        for _ in range(2):
            eng.range_sequence(dL[:nsf], dR[:nsf], d_dets, seq_offs, seq_out, seq_cnt, rect=rect_cfg,
                               stream=stream.cuda_stream)
        torch.cuda.synchronize()
        reps = 3
        t0 = time.perf_counter()
        for _ in range(reps):
            eng.range_sequence(dL[:nsf], dR[:nsf], d_dets, seq_offs, seq_out, seq_cnt, rect=rect_cfg,
                               stream=stream.cuda_stream)
        torch.cuda.synchronize()
        sdt = (time.perf_counter() - t0) / reps
        seq = {"config": f"C2 frames, {nsf} per call: offset search delta -3..3 on the central half (BM 32 disp, "
                         "9x9) + filter_offset scan + ranging of the rect-corrected pairs (rg_range_sequence)",
               "frames_per_sec": nsf / sdt, "boxes_per_sec": int(seq_cnt.sum().item()) / sdt,
               "ms_per_frame": 1000.0 * sdt / nsf}
    except Exception as e:  # pragma: no cover
        seq = {"error": str(e)}

    # ---- SGM dense baseline on the same frames: 64
    # disparities, P1 8 / P2 32 (sgm.hpp defaults), rg_sgm_frames
    sgm = None
    try:
        import ctypes as C
        nsg = min(F, 8)
        sp = rg.SgmParams(64, 0, 8, 32).to_c()
        sgm_out = torch.zeros(nsg * W * H, dtype=torch.int16, device=dev)

        def sgm_run():
            ctx.check(rg.lib().rg_sgm_frames(ctx.handle, dL.data_ptr(), dR.data_ptr(), nsg, dL.stride(0), W, W, H,
                                             C.byref(sp), sgm_out.data_ptr(), C.c_void_p(stream.cuda_stream)))
        sgm_run()
        torch.cuda.synchronize()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        sgm_run()
        g1.record(stream)
        torch.cuda.synchronize()
        sms = g0.elapsed_time(g1) / nsg
        sgm = {"config": "1920x1080 C2 frames, census SGM, 64 disparities, P1 8, P2 32, 4 paths (rg_sgm_frames)",
               "ms_per_frame": sms, "frames_per_sec": 1000.0 / sms}
    except Exception as e:  # pragma: no cover
        sgm = {"error": str(e)}

    # ---- C5: the sharded 4096-frame stream (BASELINE config 4)
    stream_c5 = None
    if args.stream_frames > 0:
        try:
            stream_c5 = c5_stream(args, eng, ctx, dev, stream, rank, world, dets, recs, offs)
        except Exception as e:  # pragma: no cover
            stream_c5 = {"error": str(e)}
        torch.cuda.empty_cache()

    # ---- C3 and 9x7 C1 (BASELINE configs 2 and 0), rank 0 only
    c3 = c1w = None
    if rank == 0 and args.c3_frames > 0:
        try:
            c3 = config_c3(args, ctx, dev, stream)
        except Exception as e:  # pragma: no cover
            c3 = {"error": str(e)}
        torch.cuda.empty_cache()
    if rank == 0 and args.c1_frames > 0:
        try:
            c1w = config_c1_9x7(args, ctx, dev, stream)
        except Exception as e:  # pragma: no cover
            c1w = {"error": str(e)}
        torch.cuda.empty_cache()

    # ---- roofline of the dominant kernel (stage times from CUDA events on our stream)
    hbm_peak, sm_max, peak_kind = peaks()
    # per step: each profiled step is one rg_range_frames call (one pipeline)
    census_ms = stage_ms[0] / roof_steps
    match_ms = stage_ms[2] / roof_steps
    census_gbs = CENSUS_BYTES_PER_FRAME * F / (census_ms / 1000.0) / 1e9
    req = census_required_bytes(dets, W, H)
    req_frame = req["bytes"]
    census_req_gbs = req_frame * F / (census_ms / 1000.0) / 1e9
    evals_per_launch = r_evals / roof_steps
    clk_mhz = clk["sm_mhz"] or sm_max
    popc_clk, popc_src = popc_peak_per_clk()
    popc_peak = popc_clk * N_SM * clk_mhz * 1e6
    match_rate = evals_per_launch / (match_ms / 1000.0)
    traffic = None
    try:  # dram read + write bytes of the census kernels of one 256-frame launch (ncu, profiles/)
        with open(os.path.join(ROOT, "profiles", "r2_traffic.json")) as f:
            tr = json.load(f)
        traffic = tr["census_dram_bytes_per_launch"] * F / tr["frames_per_launch"]
    except Exception:
        pass
    census_roof = {"bound": "hbm", "achieved": census_req_gbs, "peak": hbm_peak, "unit": "GB/s",
                   "frac": census_req_gbs / hbm_peak, "traffic": traffic,
                   "kernel": "census_rows_kernel + census_rowtile_kernel<1> (FAR ROI tiles, full raster) + "
                             "census_rowtile_kernel<2> (CLOSE ROI tiles, reduced raster)",
                   "peak_source": peak_kind, "algorithmic_bytes_per_launch": req_frame * F,
                   "algorithmic_bytes": f"the codes of the reference's ROI rectangles the matcher can read: "
                                        f"{req['codes']} 4-B codes per frame (both images, full + reduced "
                                        f"rasters) + the {req['image_bytes']} image bytes under their windows",
                   "ms_per_launch": census_ms, "frac_of_nominal_8000_gbs": census_req_gbs / 8000.0,
                   "reference_roi_equivalent": {
                       "bytes_per_launch": req["ref_bytes"] * F,
                       "effective_gbs": req["ref_bytes"] * F / (census_ms / 1000.0) / 1e9,
                       "note": f"the reference's whole ROI rectangles ({req['ref_full_codes']} full + "
                               f"{req['ref_reduced_codes']} reduced codes per image, both images read) over the "
                               "same time: an effective rate"},
                   "full_frame_kernel": {
                       "kernel": "census_pairs_kernel (batches under 12 frames, single-image API, SGM; "
                                 "here the same 256-frame steps with rg_set_census_rois(0))",
                       "frames": ff, "ms_per_launch": ff_ms,
                       "achieved_gbs": CENSUS_BYTES_PER_FRAME * ff / (ff_ms / 1000.0) / 1e9,
                       "frac": CENSUS_BYTES_PER_FRAME * ff / (ff_ms / 1000.0) / 1e9 / hbm_peak,
                       "bytes": "SURVEY 8(d): 24,883,200 B per C2 frame (both images read, full + reduced "
                                "rasters written)"},
                   "full_frame_equivalent": {
                       "bytes_per_launch": CENSUS_BYTES_PER_FRAME * F, "effective_gbs": census_gbs,
                       "note": "SURVEY 8(d) full-frame census bytes (24,883,200 per C2 frame) over the same time: "
                               "an effective rate, not traffic (the ROI census computes a fraction of the frame)"}}
    match_roof = {"bound": "int/popc", "achieved": match_rate / 1e12, "peak": popc_peak / 1e12,
                  "unit": "Tevals/s", "frac": match_rate / popc_peak, "kernel": "match_slots_warp_kernel",
                  "hamming_evals_per_launch": evals_per_launch, "ms_per_launch": match_ms,
                  "peak_source": f"{popc_src} {popc_clk:.2f} evals/clk/SM x {N_SM} SMs x {clk_mhz:.0f} MHz"}
    dominant = census_roof if census_ms >= match_ms else match_roof
    step_ms = ms_max / args.steps

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        try:
            k = min(F, ref_arm().cpu_threads() * 2)
            cpu = cpu_reference_run(L[:k], R[:k], recs[:offs[k]], offs[:k + 1], seconds=args.cpu_seconds)
        except Exception as e:  # pragma: no cover
            cpu = {"error": str(e)}

    mism = [p["frame_mismatches"] for p in (parity, (stream_c5 or {}).get("parity"), (c3 or {}).get("parity"),
                                            (c1w or {}).get("parity")) if isinstance(p, dict)]
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "boxes/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u8/u32/f64", "data": "synthetic",
            "frames_per_sec": fps, "boxes_per_frame": boxes_step / (F * world),
            "p50_latency_ms": 1000 * statistics.median(lat), "p50_latency_device_ms": 1000 * statistics.median(lat_dev),
            "latency_runs": args.latency_runs,
            "config": workload_config(F, world),
            "feed": "device-resident HBM ring, every frame rendered on the GPU by rg_render_frames_device",
            "e2e": {"value": e2e_value, "unit": "boxes/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "api": "rg_range_frames_host (pinned host frames, chunked H2D/compute/D2H)",
                    "h2d": "bytes the library moved (rg_get_transfer): detections and offsets by copy, and of "
                           "the frames only the 16-B segments of the image rows the ROI census reads, fetched "
                           "zero-copy by gather_rows_kernel",
                    "h2d_full_frame_bytes_per_step": h2d_full,
                    "records_equal_device_path": e2e_parity,
                    "bound": {"kind": "pcie_h2d", "achieved_gbs": e2e_h2d_gbs, "peak_gbs": pcie_gbs,
                              "frac": (e2e_h2d_gbs / pcie_gbs) if pcie_gbs else None,
                              "peak_source": "measured here: pinned 256 MiB host->device copies, best of 6 x 16"}},
            "gpu_launches": int(total_launches),
            "timed_batches_overflowed": bool(overflow_in_timed),
            "roofline": dominant,
            "kernels": {"census": census_roof, "matcher": match_roof,
                        "timing": f"per-stage CUDA events, median over {roof_steps} extra steps (one stream)",
                        "stage_ms_per_step": {k: v / roof_steps for k, v in
                                              zip(["census", "plan", "match", "aggregate"], stage_ms[:4])}},
            "hamming_evals_per_frame": evals / max(F * args.steps, 1),
            "parity_mismatches": int(sum(mism)) if mism else None,
            "parity": {"ring": parity},
            "autorect": rect,
            "sequence": seq,
            "sgm": sgm,
            "stream_c5": stream_c5,
            "c3": c3,
            "c1_9x7": c1w,
            "clocks": clk,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
