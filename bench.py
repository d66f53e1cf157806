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
import ctypes as C
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


# ------------------------------------------------------------------ C5 stream
def c5_stream(args, eng, ctx, dev, stream, rank, world, dets, ring_out0):
    """BASELINE config 4 (C5): a stream of N distinct C2 frames (seeds 1..N)
    sharded contiguously over the ranks (shard.shard_bounds),
    each shard rendered in HBM by the device frame source, ranged in chunks of
    --frames, and the per-box results all_gathered to every rank (NCCL).
    Strong scaling: the stream is fixed as the rank count grows.  Timed with
    CUDA events from the first chunk to the gathered results, max over ranks."""
    import torch
    import torch.distributed as dist
    from paper_2604_07980_b200 import synth as S
    from paper_2604_07980_b200.engine import OUT_DTYPE, pack_detections
    from paper_2604_07980_b200.shard import shard_bounds

    N, chunk = args.stream_frames, args.frames
    lo, hi = shard_bounds(N, rank, world)
    n, per = hi - lo, -(-N // world)
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
    recs, offs = pack_detections([dets] * chunk)
    d_dets = torch.from_numpy(recs.view(np.uint8)).to(dev)
    d_offs = torch.from_numpy(offs).to(dev)
    out = torch.zeros(per * rec, dtype=torch.uint8, device=dev)
    cnt = torch.zeros(per, dtype=torch.int32, device=dev)
    g_out = torch.zeros(world * out.numel(), dtype=torch.uint8, device=dev) if world > 1 else out
    g_cnt = torch.zeros(world * per, dtype=torch.int32, device=dev) if world > 1 else cnt

    def run():
        for c0 in range(0, n, chunk):
            c1 = min(n, c0 + chunk)
            eng.range_device(dL[c0:c1], dR[c0:c1], d_dets, d_offs[:c1 - c0 + 1], out[c0 * rec:c1 * rec], cnt[c0:c1],
                             stream=stream.cuda_stream)
        if world > 1:
            dist.all_gather_into_tensor(g_out, out)
            dist.all_gather_into_tensor(g_cnt, cnt)

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
    counts = g_cnt.view(world, per).cpu().numpy()
    boxes = int(sum(counts[r][:shard_bounds(N, r, world)[1] - shard_bounds(N, r, world)[0]].sum()
                    for r in range(world)))
    # global frame 0 (seed 1) is also frame 0 of rank 0's bench ring
    f0 = bytes(g_out[:rec].cpu().numpy()) == ring_out0 if ring_out0 is not None else None
    del dL, dR
    return {"config": f"C5: {N} distinct C2 frames (device-rendered, seeds 1..{N}, noise 2.0) sharded contiguously "
                      f"over {world} rank(s), ranged in chunks of {chunk}, per-box results all_gathered (NCCL)",
            "frames": N, "ms": ms, "frames_per_sec": N / (ms / 1e3), "boxes": boxes,
            "boxes_per_sec": boxes / (ms / 1e3), "scaling": "strong", "render_ms_per_rank": render_ms,
            "frame0_matches_ring": f0}


# ------------------------------------------------------------------ frames
def make_frames(n_distinct: int, seed0: int, noise: float = 2.0):
    """C2 frames: fixed 64-box layout, per-frame noise seed."""
    from paper_2604_07980_b200 import synth as S
    from concurrent.futures import ThreadPoolExecutor

    sc0, cfg = S.scene_c2(seed=seed0, noise=noise)
    dets = S.ground_truth_detections(sc0)

    def render(i):
        sc, _ = S.scene_c2(seed=seed0 + i, noise=noise)
        return S.render_stereo_pair(sc)

    with ThreadPoolExecutor(max_workers=2) as ex:  # renderer is itself row-parallel
        pairs = list(ex.map(render, range(n_distinct)))
    L = np.stack([p[0] for p in pairs])
    R = np.stack([p[1] for p in pairs])
    return L, R, dets, cfg


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_reference_run(L, R, dets, cfg, seconds: float, threads: int):
    """Time the reference (oracle/_ref, compiled from the reference headers) on
    the host cores, frame-parallel (SURVEY 8(d) mode iii), bounded in time."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_lib
    from paper_2604_07980_b200 import _abi
    from paper_2604_07980_b200.engine import OUT_DTYPE, pack_detections

    if oracle_lib.have_reference():
        chk, kind = oracle_lib.reference(), "reference"
    else:
        return None
    n = L.shape[0]
    recs, offs = pack_detections([dets] * n)
    c = cfg.to_c()
    out_stride = min(len(dets), cfg.max_objects)
    out = np.zeros(n * out_stride, OUT_DTYPE)
    cnt = np.zeros(n, np.int32)
    Lc, Rc = np.ascontiguousarray(L), np.ascontiguousarray(R)
    frames, wall = 0, 0.0
    boxes = 0
    while wall < seconds:
        t = chk.lib.ref_bench_estimate(Lc.ctypes.data, Rc.ctypes.data, W, H, n, recs.ctypes.data, offs.ctypes.data,
                                       C.byref(c), threads, out.ctypes.data, out_stride, cnt.ctypes.data)
        wall += t
        frames += n
        boxes += int(cnt.sum())
    res = {"value": boxes / wall, "unit": "boxes/s", "frames_per_sec": frames / wall, "cores": threads,
           "kind": kind, "sample": f"{frames} C2 frames ({n} distinct, noise 2.0) ranged by the reference's "
                                   f"estimate_object_disparities, {threads} threads x whole frames at workers=1, "
                                   f"{wall:.1f} s"}
    # the reference's stages on one frame at workers = 1 and
    # workers = nproc (median of reps): estimate_object_disparities (ROI
    # census path), census_transform x 2, and the C4 offset search
    try:
        from paper_2604_07980_b200 import synth as S
        d = (_abi.Detection * len(dets))(*[_abi.Detection(x.cx, x.cy, x.w, x.h, x.class_id, x.id) for x in dets])
        roi = _abi.Rect(*S.C4_ROI)
        bm = S.c4_bm().to_c()
        detail = {}
        for wk, reps, rr in ((1, 3, 1), (threads, 5, 2)):
            t = (C.c_double * 3)()
            chk.lib.ref_bench_stages.restype = C.c_int
            st = chk.lib.ref_bench_stages(C.c_void_p(Lc[0].ctypes.data), C.c_void_p(Rc[0].ctypes.data), W, H,
                                          C.byref(d), len(dets), C.byref(c), wk, reps, C.byref(roi), -8, 8,
                                          C.byref(bm), rr, t)
            if st == 0:
                detail[f"workers_{wk}"] = {"estimate_ms_per_frame": 1e3 * t[0], "census_x2_ms": 1e3 * t[1],
                                           "autorect_c4_ms": 1e3 * t[2]}
        res["stages_one_frame"] = detail
    except Exception as e:  # pragma: no cover
        res["stages_one_frame"] = f"error: {e}"
    return res


# ------------------------------------------------------------------ reference arm
def run_reference(args):
    """Reference arm: the reference's own estimate_object_disparities (compiled
    in place into oracle/_ref) on all host threads, one whole C2 frame per
    thread per step (frame-parallel), K timed steps after W warm-up steps."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_lib
    from paper_2604_07980_b200.engine import OUT_DTYPE, pack_detections

    if not oracle_lib.have_reference():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libranger_ref.so not built"}))
        return 0
    threads = cpu_threads()
    L, R, dets, cfg = make_frames(threads, 1)
    chk = oracle_lib.reference()
    recs, offs = pack_detections([dets] * threads)
    c = cfg.to_c()
    out_stride = min(len(dets), cfg.max_objects)
    out = np.zeros(threads * out_stride, OUT_DTYPE)
    cnt = np.zeros(threads, np.int32)
    Lc, Rc = np.ascontiguousarray(L), np.ascontiguousarray(R)
    secs = []
    for i in range(args.warmup + args.steps):
        t = chk.lib.ref_bench_estimate(Lc.ctypes.data, Rc.ctypes.data, W, H, threads, recs.ctypes.data,
                                       offs.ctypes.data, C.byref(c), threads, out.ctypes.data, out_stride,
                                       cnt.ctypes.data)
        if i >= args.warmup:
            secs.append(t)
    boxes = int(cnt.sum())
    total = sum(secs)
    val = boxes * len(secs) / total
    sample = (f"{threads} C2 frames per step (noise 2.0), one per host thread at workers=1 (frame-parallel), "
              f"reference estimate_object_disparities from oracle/_ref, {len(secs)} steps, {total:.1f} s")
    line = {
        "metric": METRIC, "impl": "reference", "value": val, "unit": "boxes/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * total / len(secs),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8/u32/f64",
        "data": "synthetic", "frames_per_sec": threads * len(secs) / total,
        "config": {"workload": "C2: 1920x1080 stereo, 64 boxes (48 FAR + 16 CLOSE), dx_max 256, "
                               "fwd-bwd + sub-pixel, noise 2.0", "frames_per_step": threads},
        "cpu_baseline": {"value": val, "unit": "boxes/s", "cores": threads, "kind": "reference", "sample": sample},
        "e2e": {"value": val, "unit": "boxes/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


# ------------------------------------------------------------------ our arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--frames", type=int, default=256, help="frames per step per GPU")
    ap.add_argument("--distinct", type=int, default=32, help="distinct host-rendered frames in the HBM ring "
                    "(--frame-source host)")
    ap.add_argument("--stream-frames", type=int, default=4096,
                    help="C5: frames in the sharded stream measurement (0: skip)")
    ap.add_argument("--frame-source", choices=["device", "host"], default="device",
                    help="device: every ring frame rendered on the GPU (rg_render_frames_device); "
                    "host: --distinct host renders tiled")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--latency-runs", type=int, default=300)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    os.environ["RG_DEVICE"] = str(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_2604_07980_b200 import ranger as rg
    from paper_2604_07980_b200.engine import DET_DTYPE, OUT_DTYPE, FrameEngine, pack_detections
    from paper_2604_07980_b200 import synth as S

    F = args.frames
    ctx = rg.Context(local)
    dev = torch.device("cuda", local)
    seed0 = 1 + rank * 100003
    if args.frame_source == "device":
        # every frame of the HBM ring distinct, rendered in place by the device
        # frame source (byte-identical to the host renderer, tests/test_gpu_render.py)
        args.distinct = F
        scenes = [S.scene_c2(seed=seed0 + i, noise=2.0)[0] for i in range(F)]
        dets, cfg = S.ground_truth_detections(scenes[0]), S.scene_c2(seed=seed0)[1]
        dL = torch.empty((F, H, W), dtype=torch.uint8, device=dev)
        dR = torch.empty_like(dL)
        S.render_frames_device(ctx, scenes, dL, dR)
        torch.cuda.synchronize()
        L, R = dL.cpu().numpy(), dR.cpu().numpy()  # host copies: e2e feed, CPU baseline, spot check
        idx = np.arange(F)
    else:
        L, R, dets, cfg = make_frames(args.distinct, seed0)
        # HBM ring: F frames (> L2 in bytes), tiled from the distinct renders
        idx = np.arange(F) % args.distinct
        dL = torch.from_numpy(L[idx]).to(dev)
        dR = torch.from_numpy(R[idx]).to(dev)
    n_boxes = len(dets)
    eng = FrameEngine(W, H, cfg, n_boxes, S.F_PX, S.BASELINE_M, ctx=ctx)
    recs, offs = pack_detections([dets] * F)
    d_dets = torch.from_numpy(recs.view(np.uint8)).to(dev)
    d_offs = torch.from_numpy(offs).to(dev)
    d_out = torch.zeros(F * eng.out_stride * OUT_DTYPE.itemsize, dtype=torch.uint8, device=dev)
    d_cnt = torch.zeros(F, dtype=torch.int32, device=dev)
    gather = torch.zeros(world * d_out.numel(), dtype=torch.uint8, device=dev) if world > 1 else None
    # a real (non-legacy-default) stream: the library launches on it and the
    # CUDA events below are recorded on it
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)

    def step():
        eng.range_device(dL, dR, d_dets, d_offs, d_out, d_cnt, stream=stream.cuda_stream)
        if world > 1:  # per-box results -> every rank's slab on rank 0 (NCCL over NVLink)
            dist.all_gather_into_tensor(gather, d_out)

    # ---- warmup
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    # parity spot check of the bench frames against the C oracle (frame 0)
    spot = None
    if rank == 0:
        try:
            sys.path.insert(0, os.path.join(ROOT, "tests"))
            import oracle_lib
            from paper_2604_07980_b200 import _abi
            want, _ = oracle_lib.oracle().estimate(L[0], R[0], [_abi.Detection(d.cx, d.cy, d.w, d.h, d.class_id, d.id)
                                                                for d in dets], cfg.to_c(), S.F_PX, S.BASELINE_M)
            got = np.frombuffer(d_out.cpu().numpy().tobytes(), OUT_DTYPE)[:int(d_cnt[0])]
            spot = bool(len(got) == len(want) and all(bytes(w) == got[i].tobytes() for i, w in enumerate(want)))
        except Exception as e:  # pragma: no cover
            spot = f"error: {e}"

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
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    clk = clocks.stop()
    _, _, total_launches = ctx.counters()
    evals, blocks = ctx.work()
    # ---- kernel rooflines: the same steps with per-stage CUDA events
    ctx.reset_counters()
    ctx.set_overlap(False)
    ctx.set_profiling(True)
    roof_steps = max(3, min(args.steps, 10))
    for _ in range(roof_steps):
        step()
    torch.cuda.synchronize()
    ctx.set_profiling(False)
    ctx.set_overlap(True)
    stage_ms, stage_launches, _ = ctx.counters()
    r_evals, _ = ctx.work()
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    boxes_step = int(d_cnt.sum().item())
    total_boxes = boxes_step * args.steps * world
    value = total_boxes / (ms_max / 1000.0)
    fps = F * args.steps * world / (ms_max / 1000.0)

    # ---- end-to-end through the public host API (pinned host frames, H2D/D2H inside)
    keep = []

    def pin(a):  # pinned host copy of any numpy array (structured dtypes included)
        t = torch.empty(a.nbytes, dtype=torch.uint8).pin_memory()
        keep.append(t)
        v = t.numpy().view(a.dtype).reshape(a.shape)
        v[...] = a
        return v
    hL, hR = pin(L[idx]), pin(R[idx])
    h_recs, h_offs = pin(recs), pin(offs)
    h_out = pin(np.zeros(F * eng.out_stride, OUT_DTYPE))
    h_cnt = pin(np.zeros(F, np.int32))
    for _ in range(2):
        eng.range_host(hL, hR, h_recs, h_offs, h_out, h_cnt, chunk=32, stream=stream.cuda_stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    e2e_steps = max(2, args.steps // 2)
    for _ in range(e2e_steps):
        eng.range_host(hL, hR, h_recs, h_offs, h_out, h_cnt, chunk=32, stream=stream.cuda_stream)
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    te = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = int(h_cnt.sum()) * e2e_steps * world / float(te.item())
    h2d = int(hL.nbytes + hR.nbytes + h_recs.nbytes + h_offs.nbytes)
    d2h = int(h_out.nbytes + h_cnt.nbytes)
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
        eng.range_host(hL[i % F:i % F + 1], hR[i % F:i % F + 1], h_recs[:n_boxes], h_offs[:2] - 0, h_out[:eng.out_stride],
                       h_cnt[:1], chunk=1, stream=stream.cuda_stream)
        lat.append(time.perf_counter() - a)
    lat_dev = []
    for i in range(max(50, args.latency_runs // 3)):
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
            rec0 = eng.out_stride * OUT_DTYPE.itemsize
            # ring frame 0 again (the latency runs reused the first output slot)
            eng.range_device(dL[0:1], dR[0:1], d_dets, d_offs[:2], d_out, d_cnt, stream=stream.cuda_stream)
            torch.cuda.synchronize()
            stream_c5 = c5_stream(args, eng, ctx, dev, stream, rank, world, dets,
                                  bytes(d_out[:rec0].cpu().numpy()) if rank == 0 else None)
        except Exception as e:  # pragma: no cover
            stream_c5 = {"error": str(e)}
        torch.cuda.empty_cache()

    # ---- roofline of the dominant kernel (stage times from CUDA events on our stream)
    hbm_peak, sm_max, peak_kind = peaks()
    census_ms = stage_ms[0] / max(stage_launches[0], 1)
    match_ms = stage_ms[2] / max(stage_launches[2], 1)
    census_gbs = CENSUS_BYTES_PER_FRAME * F / (census_ms / 1000.0) / 1e9
    evals_per_launch = r_evals / max(stage_launches[2], 1)
    clk_mhz = clk["sm_mhz"] or sm_max
    popc_clk, popc_src = popc_peak_per_clk()
    popc_peak = popc_clk * N_SM * clk_mhz * 1e6
    match_rate = evals_per_launch / (match_ms / 1000.0)
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            tr = json.load(f)
        traffic = tr.get("census_bytes_per_frame", None)
        traffic = traffic * F if traffic else None
    except Exception:
        pass
    census_roof = {"bound": "hbm", "achieved": census_gbs, "peak": hbm_peak, "unit": "GB/s",
                   "frac": census_gbs / hbm_peak, "traffic": traffic, "kernel": "census_pairs_kernel",
                   "peak_source": peak_kind, "algorithmic_bytes_per_launch": CENSUS_BYTES_PER_FRAME * F,
                   "ms_per_launch": census_ms, "frac_of_nominal_8000_gbs": census_gbs / 8000.0}
    match_roof = {"bound": "int/popc", "achieved": match_rate / 1e12, "peak": popc_peak / 1e12,
                  "unit": "Tevals/s", "frac": match_rate / popc_peak, "kernel": "match_slots_warp_kernel",
                  "hamming_evals_per_launch": evals_per_launch, "ms_per_launch": match_ms,
                  "peak_source": f"{popc_src} {popc_clk:.2f} evals/clk/SM x {N_SM} SMs x {clk_mhz:.0f} MHz"}
    dominant = census_roof if census_ms >= match_ms else match_roof
    step_ms = ms_max / args.steps

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        try:
            cpu = cpu_reference_run(L[:min(args.distinct, cpu_threads() * 2)], R[:min(args.distinct, cpu_threads() * 2)],
                                    dets, cfg, seconds=args.cpu_seconds, threads=cpu_threads())
        except Exception as e:  # pragma: no cover
            cpu = {"error": str(e)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "boxes/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u8/u32/f64", "data": "synthetic",
            "frames_per_sec": fps, "boxes_per_frame": boxes_step / F,
            "p50_latency_ms": 1000 * statistics.median(lat), "p50_latency_device_ms": 1000 * statistics.median(lat_dev),
            "config": {"workload": "C2: 1920x1080 rendered stereo pairs, 64 boxes (48 FAR + 16 CLOSE), "
                                   "dx_max_far = dx_max_close = 256, tau_v 1.0, fwd-bwd + sub-pixel, range z",
                       "frames_per_step_per_gpu": F, "distinct_frames": args.distinct, "frame_source": args.frame_source,
                       "noise_sigma": 2.0,
                       "l2": f"inputs {2 * F * W * H / 1e6:.0f} MB + census {F * CENSUS_BYTES_PER_FRAME / 1e6:.0f} MB "
                             f"per step > 126 MB L2 (no flush needed)",
                       "parallelism": f"frame-sharded dp{world}, NCCL all_gather of per-box results"},
            "e2e": {"value": e2e_value, "unit": "boxes/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "api": "rg_range_frames_host (pinned host frames, chunked H2D/compute/D2H)",
                    "bound": {"kind": "pcie_h2d", "achieved_gbs": e2e_h2d_gbs, "peak_gbs": pcie_gbs,
                              "frac": (e2e_h2d_gbs / pcie_gbs) if pcie_gbs else None,
                              "peak_source": "measured here: pinned 256 MiB host->device copies, best of 6 x 16"}},
            "gpu_launches": int(total_launches),
            "roofline": dominant,
            "kernels": {"census": census_roof, "matcher": match_roof,
                        "timing": f"per-stage CUDA events over {roof_steps} extra steps (one stream)",
                        "stage_ms_per_step": {k: v / roof_steps for k, v in
                                              zip(["census", "plan", "match", "aggregate"], stage_ms[:4])}},
            "hamming_evals_per_frame": evals / max(F * args.steps, 1),
            "autorect": rect,
            "sequence": seq,
            "sgm": sgm,
            "stream_c5": stream_c5,
            "clocks": clk,
            "parity_spot_check_vs_oracle": spot,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
