"""Benchmark: megapixels/s of (pre-integration + space-variant filter).

python bench.py [--gpus N] [--steps K] [--warmup W] [--config 3] [--orders 1,2,3,4] [--impl reference]
python bench.py --config 4 [--frames 64 | --frames-per-gpu F] --steps 1   (frames sharded over GPUs)
python bench.py --config 5 --steps 1                                      (one image, row strips, NCCL halos)

Default workload: BASELINE.json configs[2], the largest single-GPU config
(c3_4096_u8_grid32: 4096^2 u8, sigma_major U[2,40], ratio U[1,6] on an
upsampled 32^2 grid), "orders 1..4 swept".  The JSON line's headline is the
first order (order 1: the paper's own 16-tap filter, Alg. 3); every order's
numbers (value, roofline, cpu_baseline, e2e) are under "orders".

One step = one pass of the whole hot path over the image, inputs resident in
HBM:
  * order 1 (global mode): bsf_preintegrate_exact (the paper's
    single global pre-integration, exact int64) + bsf_filter_exact (per-pixel
    finite difference with an exact integer contraction of Eq. (11));
  * orders 2-3: bsf_run on the tile-anchored fused kernel (running sums per
    super-tile, exact split contraction on the FP64 tensor cores);
  * order 4: bsf_run_tiles on a fixed sample of whole anchoring tiles (16 per
    SM: the four corners + uniform; the double-double tile kernel: a full
    4096^2 image takes ~200 s at order 4, profiles/r02_order4_full.json --
    PAPER.md:161-166; the sample is stated in the line).
Orders 3 and 4 take min(K, 2) and 1 timed steps after one warm-up step (their
steps take seconds); orders 1-2 take K steps after W >= 3 warm-ups.  The L2
(126 MB) is flushed between timed steps (256 MB write, untimed); each step is
timed with CUDA events on the launching stream.  For N > 1 (torchrun, one rank
per GPU) every rank filters its own frame of the config (independent images:
weak scaling); time = max over ranks.

--impl reference times the CPU oracle (the deliberately slow reference arm of
this tier) on bounded pixel samples of the same workload, on rank 0 only.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402

METRIC = "megapixels/sec (pre-integration + space-variant filter)"
UNIT = "Mpx/s"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


def _json(path):
    with open(os.path.join(ROOT, path)) as fh:
        return json.load(fh)


def _src_hash():
    """Hash of the CUDA sources: a committed ncu traffic figure is only reported
    for the build it was captured on."""
    h = hashlib.sha1()
    d = os.path.join(ROOT, "paper_1109_5114_b200", "csrc")
    for f in sorted(os.listdir(d)):
        with open(os.path.join(d, f), "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()[:12]


def _traffic(workload, order, kernel):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel` from
    the committed ncu --set full capture (profiles/r02_traffic.json), if it was
    taken on these exact sources; else None."""
    try:
        t = _json("profiles/r02_traffic.json")
        e = t["captures"]["%s/r%d/%s" % (workload, order, kernel)]
        return e["dram_bytes"] if e["src_hash"] == _src_hash() else None
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + q,
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 3 + i and r[3 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def _sample_pixels(w, n, seed):
    """Stratified pixels for the CPU legs (corners and edges, min/max sigma, the
    rest uniform): the method-independent strata of BASELINE.md's plan (the
    clamp/zero-scale/sector strata need the method and are sampled by the
    GPU tests, tests/strata.py)."""
    H, W = w.height, w.width
    rng = np.random.default_rng(seed)
    pts = [(0, 0), (W - 1, 0), (0, H - 1), (W - 1, H - 1), (W // 2, 0), (0, H // 2), (W - 1, H // 2),
           (W // 2, H - 1)]
    pool_x = rng.integers(0, W, 4000)
    pool_y = rng.integers(0, H, 4000)
    c = synth.cov_at(w, pool_x, pool_y).numpy()
    smaj = np.maximum(c[0], c[1])
    o = np.argsort(smaj)
    k = max(1, n // 8)
    pts += list(zip(pool_x[o[:k]], pool_y[o[:k]])) + list(zip(pool_x[o[-k:]], pool_y[o[-k:]]))
    while len(pts) < n:
        pts.append((int(rng.integers(0, W)), int(rng.integers(0, H))))
    pts = pts[:n]
    rng.shuffle(pts)
    xs = np.array([p[0] for p in pts], dtype=np.int64)
    ys = np.array([p[1] for p in pts], dtype=np.int64)
    return xs, ys


_IMG = {}


def _oracle_chunk(w, r, xs, ys, nthreads):
    """The oracle at pixels (xs, ys), OpenMP-parallel over the pixels: the image
    and covariance are exactly what the GPU consumes (synth values)."""
    import oracle as O
    key = (w.name, w.seed)
    if key not in _IMG:
        _IMG.clear()
        _IMG[key] = synth.make_image(w).numpy()
    cov = synth.cov_at(w, xs, ys).numpy().astype(np.float64)
    return O.filter_points(_IMG[key], xs, ys, cov[0], cov[1], cov[2], policy=w.basis, r=r, nthreads=nthreads)[0]


def cpu_baseline(w, r, budget_s: float, max_points: int, seed=12):
    """The oracle as it stands, on a bounded stratified sample of the workload;
    the full-image time is extrapolated (labelled so)."""
    nthreads = os.cpu_count() or 1
    xs, ys = _sample_pixels(w, max_points, seed)
    _oracle_chunk(w, r, xs[:1], ys[:1], 1)  # image generation outside the timed sample
    done, t0 = 0, time.perf_counter()
    while done < max_points and time.perf_counter() - t0 < budget_s:
        sl = slice(done, min(done + nthreads, max_points))
        _oracle_chunk(w, r, xs[sl], ys[sl], nthreads)
        done = sl.stop
    dt = time.perf_counter() - t0
    v = done / dt / 1e6
    return {"value": v, "unit": UNIT, "cores": nthreads, "kind": "oracle",
            "sample": "%d stratified pixels of %s at order %d in %.2f s (direct sum, exact box-spline kernel, "
                      "OpenMP over the pixels)" % (done, w.name, r, dt),
            "full_image_s_extrapolated": w.width * w.height / (v * 1e6) if v > 0 else None}


def run_reference(args, w, orders):
    """CPU oracle arm: bounded stratified samples of the workload per step."""
    nthreads = os.cpu_count() or 1
    r = orders[0]
    per_step = args.ref_points
    if per_step <= 0:  # auto: ~0.5 s of oracle work per step (calibrated on a separate stratified sample)
        cx, cy = _sample_pixels(w, 2 * nthreads, 13)
        _oracle_chunk(w, r, cx[:1], cy[:1], 1)  # image generation outside the calibration
        t0 = time.perf_counter()
        _oracle_chunk(w, r, cx, cy, nthreads)
        per_px = (time.perf_counter() - t0) / len(cx)
        per_step = int(min(4000, max(nthreads, 0.5 / max(per_px, 1e-9))))
    xs, ys = _sample_pixels(w, per_step * (args.steps + args.warmup), 11)

    def step(i):
        sl = slice(i * per_step, (i + 1) * per_step)
        _oracle_chunk(w, r, xs[sl], ys[sl], nthreads)

    _oracle_chunk(w, r, xs[:1], ys[:1], 1)  # image generation outside the timed region
    for i in range(args.warmup):
        step(i)
    t0 = time.perf_counter()
    for i in range(args.steps):
        step(args.warmup + i)
    dt = time.perf_counter() - t0
    value = per_step * args.steps / dt / 1e6
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": w.name, "order": r, "width": w.width, "height": w.height,
                       "basis": "dual", "in_dtype": w.in_dtype,
                       "impl": "oracle: fp64 direct sum with the exact box-spline kernel"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": nthreads, "kind": "oracle",
                             "sample": "%d stratified pixels per step of %s at order %d" % (per_step, w.name, r)},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def _tile_sample(w, unit, n, seed=21):
    """A fixed stratified sample of whole anchoring tiles (order 4): a spread of
    tile rows/columns, the four corners, and the tiles of the largest and
    smallest sigma."""
    ntx, nty = (w.width + unit - 1) // unit, (w.height + unit - 1) // unit
    rng = np.random.default_rng(seed)
    tx = list(rng.integers(0, ntx, n))
    ty = list(rng.integers(0, nty, n))
    tx[:4] = [0, ntx - 1, 0, ntx - 1]
    ty[:4] = [0, 0, nty - 1, nty - 1]
    ids = sorted({int(b * ntx + a) for a, b in zip(tx, ty)})
    return torch.tensor(ids, dtype=torch.int32)


def time_order(args, w, r, dev, rank, world, stream, flush, pg):
    """Time one order of the workload; returns the per-order result dict."""
    from paper_1109_5114_b200 import bsf
    plan = bsf.Plan(w.width, w.height, batch=1, channels=1,
                    in_dtype=bsf.BSF_U8 if w.in_dtype == "u8" else bsf.BSF_F32, out_dtype=bsf.BSF_F64,
                    order=r, basis=w.basis, max_sigma=w.max_sigma, precision=bsf.BSF_PREC_DD, device=dev.index,
                    anchor=bsf.BSF_ANCHOR_AUTO)
    geo = plan.geometry
    img = synth.make_image(w, frame=rank, device=dev).contiguous()
    cov = synth.make_cov(w, device=dev).contiguous()
    out = torch.empty((1, w.height, w.width), dtype=torch.float64, device=dev)
    npx = w.width * w.height
    mode = "global" if geo.global_mode else ("tile" if r <= 3 else "tiles_sample")
    K = args.steps if r <= 2 else (min(args.steps, 2) if r == 3 else 1)
    Wm = max(3, args.warmup)  # W >= 3 at every order (orders 3 / 4: ~5 s per step)
    g = plan.empty_g_exact() if mode == "global" else None
    tiles = None
    if mode == "tiles_sample":
        tiles = _tile_sample(w, geo.tile_unit, args.r4_tiles).to(dev)
        npx = int(tiles.numel()) * geo.tile_unit * geo.tile_unit

    def step(ev=None):
        if mode == "global":
            plan.preintegrate_exact(img, g, stream)
            if ev is not None:
                ev.record(stream)
            plan.filter_exact(g, cov, out, stream)
        elif mode == "tile":
            if ev is not None:
                ev.record(stream)
            plan.run(img, cov, out, stream)
        else:
            if ev is not None:
                ev.record(stream)
            plan.run_tiles(img, cov, out, tiles, stream)

    for _ in range(Wm):
        step()
        flush.zero_()
    torch.cuda.synchronize()
    plan.stats(reset=True)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    mids = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    launches0 = plan.launch_count()
    if pg:
        pg.barrier()
    torch.cuda.synchronize()
    for i in range(K):
        starts[i].record(stream)
        step(mids[i])
        ends[i].record(stream)
        flush.zero_()
    torch.cuda.synchronize()
    if pg:
        pg.barrier()
    launches = plan.launch_count() - launches0
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    kern_ms = [m.elapsed_time(e) for m, e in zip(mids, ends)]
    pre_ms = [s.elapsed_time(m) for s, m in zip(starts, mids)]
    ms = sum(step_ms) / K
    kms = sum(kern_ms) / K
    pms = sum(pre_ms) / K
    stats = plan.stats(reset=True)
    if pg:
        t = torch.tensor([ms], device=dev)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        ms = float(t[0])
    value = world * npx / (ms * 1e-3) / 1e6
    res = {"value": value, "ms_per_step": ms, "steps": K, "warmup": Wm, "mode": mode, "pixels_per_step": npx,
           "gpu_launches": launches, "launches_per_step": launches / K,
           "stats": {k: stats[k] for k in ("pixels", "clamped", "zero_scale", "theta_prime", "flags",
                                           "double_double", "macs")}}
    if mode == "tiles_sample":
        res["sample"] = ("%d whole %dx%d anchoring tiles (%.2f %% of the image; corners + uniform) through "
                         "bsf_run_tiles" % (tiles.numel(), geo.tile_unit, geo.tile_unit,
                                            100.0 * npx / (w.width * w.height)))
    # --- e2e: bsf_run_host (pinned host buffers, copies inside the timed region)
    if mode != "tiles_sample":
        f_h = img.cpu().pin_memory()
        c_h = cov.cpu().pin_memory()
        o_h = torch.empty(out.shape, dtype=out.dtype).pin_memory()
        plan.run_host(f_h, c_h, o_h, stream)
        torch.cuda.synchronize()
        Ke = min(K, 3)
        e_s = [torch.cuda.Event(enable_timing=True) for _ in range(Ke)]
        e_e = [torch.cuda.Event(enable_timing=True) for _ in range(Ke)]
        if pg:
            pg.barrier()
        for i in range(Ke):
            e_s[i].record(stream)
            plan.run_host(f_h, c_h, o_h, stream)
            e_e[i].record(stream)
            flush.zero_()
        torch.cuda.synchronize()
        e2e_ms = sum(a.elapsed_time(b) for a, b in zip(e_s, e_e)) / Ke
        if pg:
            t = torch.tensor([e2e_ms], device=dev)
            pg.all_reduce(t, op=pg.ReduceOp.MAX)
            e2e_ms = float(t[0])
        res["e2e"] = {"value": world * npx / (e2e_ms * 1e-3) / 1e6, "unit": UNIT, "steps": Ke,
                      "h2d_bytes_per_step": f_h.numel() * f_h.element_size() + c_h.numel() * c_h.element_size(),
                      "d2h_bytes_per_step": o_h.numel() * o_h.element_size()}
    else:
        res["e2e"] = None
    res["roofline"] = roofline(w, r, mode, plan, stats, npx, kms, pms, ms)
    return res


def roofline(w, r, mode, plan, stats, npx, kms, pms, ms):
    peaks, src = _peaks()
    sm_mhz = peaks.get("sm_max_mhz", 1965.0)
    nsm = torch.cuda.get_device_properties(0).multi_processor_count
    geo = plan.geometry
    in_b = 1 if w.in_dtype == "u8" else 4
    if mode == "global":
        # dominant kernel: the order-1 integer gather.  Algorithmic work = the
        # exact contraction of Eq. (11): window x monomials multiply-adds per
        # tap (counted by the kernel, bsf_stats.macs), each an int64 x int8
        # product done as 3 int32 limb multiply-adds (no rounding).  Peak: the
        # int32 multiply-add rate: IMAD issues on the FMA pipe at a reciprocal
        # throughput of 2 cycles per warp instruction per SMSP
        # (B300_MICROARCH.md, 'Pipe rates'), i.e. 64 lanes/clk/SM.
        imad = 3.0 * stats["macs"] / max(stats["pixels"], 1) * npx
        achieved = imad / (kms * 1e-3) / 1e12
        peak = nsm * 64 * sm_mhz * 1e6 / 1e12
        g_bytes = geo.nbases * geo.g_height * geo.g_width * 8 * (npx // (w.width * w.height))
        pre_bytes = npx * in_b + g_bytes  # read f once, write g once
        gat_bytes = g_bytes + npx * (12 + 8)  # read g once (taps from L2), cov 3 x f32, out f64
        hbm = peaks.get("hbm_gbs", 6650.0)
        fma = stats["macs"] / max(stats["pixels"], 1)  # window x monomials per tap
        roof = {"bound": "alu", "kernel": "gx1_kernel (order-1 exact integer gather)",
                "achieved": achieved, "peak": peak, "unit": "Tintop/s", "frac": achieved / peak,
                "traffic": _traffic(w.name, r, "gx1_kernel"),
                "peak_source": "%d SM x 64 int32 multiply-adds/clk (IMAD on the FMA pipe, 2 cycles per warp "
                               "instruction per SMSP: B300_MICROARCH.md) x %.0f MHz (sm_max, %s)" % (nsm, sm_mhz, src),
                "algorithmic": "3 int32 limb multiply-adds per (tap, window slot, monomial): %.0f per px" % (
                    imad / npx),
                "kernel_ms": kms, "share_of_step": kms / ms if ms else None,
                # the same kernel against the other two rooflines SURVEY.md 8(d) names
                "hbm": {"algorithmic_bytes": gat_bytes, "achieved_gbs": gat_bytes / (kms * 1e-3) / 1e9,
                        "peak_gbs": hbm, "frac": gat_bytes / (kms * 1e-3) / 1e9 / hbm},
                "fp64_fma_equiv": {"fma_per_px": fma, "achieved_tfma": fma * npx / (kms * 1e-3) / 1e12,
                                   "peak_tfma": _json("profiles/r01_fp64_peak.json")["fp64_fma_peak_tflops"] / 2,
                                   "frac": fma * npx / (kms * 1e-3) / 1e12 /
                                   (_json("profiles/r01_fp64_peak.json")["fp64_fma_peak_tflops"] / 2)},
                "step_hbm": {"algorithmic_bytes": pre_bytes + gat_bytes,
                             "achieved_gbs": (pre_bytes + gat_bytes) / (ms * 1e-3) / 1e9 if ms else None,
                             "frac": (pre_bytes + gat_bytes) / (ms * 1e-3) / 1e9 / hbm if ms else None},
                "preintegration": {"bound": "hbm", "kernel": "scan_row_kernel / scan_strip_tma_kernel "
                                   "(TMA-fed rows; int64, 4 levels per basis)", "ms": pms, "algorithmic_bytes": pre_bytes,
                                   "achieved_gbs": pre_bytes / (pms * 1e-3) / 1e9, "peak_gbs": hbm,
                                   "frac": pre_bytes / (pms * 1e-3) / 1e9 / hbm,
                                   "traffic": _traffic(w.name, r, "scan")}}
        pt = roof["preintegration"]["traffic"]
        # the bytes the 8 level launches actually move (one read + one write
        # of an int64 plane per level, ncu) over the same measured time
        roof["preintegration"]["traffic_frac"] = pt / (pms * 1e-3) / 1e9 / hbm if pt else None
        return roof
    if mode == "tile" and plan.uses_fused():
        fp = _json("profiles/r01_fp64_peak.json")
        macs_px = stats["macs"] / max(stats["pixels"], 1)
        achieved = 2.0 * macs_px * npx / (kms * 1e-3) / 1e12
        return {"bound": "tensor", "pipe": "FP64 tensor (DMMA m8n8k4; tcgen05 has no f64 kind)",
                "kernel": "fused_kernel<%d> (per-super-tile pre-integration + exact split contraction)" % r,
                "achieved": achieved, "peak": fp["fp64_tensor_peak_tflops"], "unit": "TFLOP/s",
                "frac": achieved / fp["fp64_tensor_peak_tflops"], "traffic": _traffic(w.name, r, "fused_kernel"),
                "peak_source": "measured: tools/fp64_peak.cu DMMA m8n8k4 (profiles/r01_fp64_peak.json)",
                "algorithmic": "2 x interpolation multiply-adds of Eq. (11) (window x monomials per tap, counted "
                               "by the kernel): %.0f MAC/px" % macs_px,
                "executed_limbs": 2 if r <= 2 else 3, "kernel_ms": kms, "share_of_step": kms / ms if ms else None}
    # order 4: the double-double tile kernel; algorithmic FMA per pixel (SURVEY
    # C.2): (r+1)^ns taps x window x (monomials + 1) for the weights' Horner
    from paper_1109_5114_b200 import lut
    tp = stats["theta_prime"] / max(stats["pixels"], 1)
    zs = stats["zero_scale"] / max(stats["pixels"], 1)
    fma = 0.0
    for b, fb in ((0, 1 - tp), (1, tp)):
        T = lut.load(b, r)["variants"]
        full = (r + 1) ** 4 * float(np.mean(T[0]["counts"])) * (T[0]["nmon"] + 1)
        var = (r + 1) ** 3 * float(np.mean(T[1]["counts"])) * (T[1]["nmon"] + 1)
        fma += fb * ((1 - zs) * full + zs * var)
    achieved = 2 * fma * npx / (kms * 1e-3) / 1e12
    peak = _json("profiles/r01_fp64_peak.json")["fp64_fma_peak_tflops"]
    return {"bound": "alu", "kernel": "tile_kernel<4, dd> (per-tile pre-integration + double-double mesh)",
            "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
            "traffic": _traffic(w.name, r, "tile_kernel"),
            "peak_source": "measured: tools/fp64_peak.cu DFMA (profiles/r01_fp64_peak.json)",
            "algorithmic": "(r+1)^ns taps x mean window x (monomials + 1) FMA per px (SURVEY.md C.2), weighted by "
                           "the measured basis / zero-scale mix: %.3g FMA/px" % fma,
            "kernel_ms": kms, "share_of_step": kms / ms if ms else None}


def run_partitioned(args, rank, world, local):
    """Configs 4 and 5 (BASELINE.json: frames sharded over GPUs; one image in
    row strips with NCCL halo exchange), one process per GPU.  Config 4: the
    frames (3 channels each, one covariance field per frame) are split over
    the ranks (parallel.shard_range), no collective on the data path (weak in
    frames per rank when --frames grows with N; strong at a fixed --frames).
    Config 5: one multi-GPU plan per rank (bsf_plan_desc rank / nranks /
    nccl_id), created once; bsf_run exchanges the input halo rows with
    ncclSend/ncclRecv inside the library and filters the strip's own rows
    (strong scaling).  Time: barrier + synchronize around the timed steps,
    CUDA events on the launching stream, max over ranks."""
    from paper_1109_5114_b200 import bsf
    from paper_1109_5114_b200 import parallel as PL
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    w = synth.workload(args.config)
    if args.config == 4:
        f0, f1 = PL.shard_range(args.frames, rank, world)
        nf, C = f1 - f0, w.channels
        plan = bsf.Plan(w.width, w.height, batch=max(nf, 1), channels=C, in_dtype=bsf.BSF_F32, order=w.order,
                        basis=w.basis, max_sigma=w.max_sigma, anchor=bsf.BSF_ANCHOR_TILE, device=local)
        img = torch.stack([synth.make_image(w, frame=f, channel=c, device=dev) for f in range(f0, f1)
                           for c in range(C)]).contiguous() if nf else None
        cov = torch.stack([synth.make_cov(w, frame=f, device=dev) for f in range(f0, f1)]).contiguous() if nf \
            else None
        out = torch.empty((max(nf, 1) * C, w.height, w.width), dtype=torch.float64, device=dev)
        npx_rank = nf * C * w.width * w.height

        def step():
            if nf:
                plan.run(img, cov, out)
        cfg = {"workload": w.name, "order": w.order, "frames": args.frames, "channels": C, "frames_per_rank": nf,
               "parallelism": "frames sharded over %d ranks (no data-path collective)" % world}
        scaling = "weak" if args.frames_per_gpu else "strong"
    else:
        H = w.height
        nid = None
        if world > 1:
            obj = [bsf.get_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            nid = obj[0]
        plan = bsf.Plan(w.width, H, in_dtype=bsf.BSF_F32, order=w.order, basis=w.basis, max_sigma=w.max_sigma,
                        anchor=bsf.BSF_ANCHOR_TILE, device=local, rank=rank, nranks=world, nccl_id=nid)
        g = plan.geometry
        y0, y1 = g.row0, g.row0 + g.row_count
        f_own = synth.make_image(w, window=(y0, y1, 0, w.width), device=dev)[None].contiguous()
        cov_own = synth.make_cov(w, window=(y0, y1, 0, w.width), device=dev).contiguous()
        out = torch.empty((1, y1 - y0, w.width), dtype=torch.float64, device=dev)
        npx_rank = (y1 - y0) * w.width

        def step():
            plan.run(f_own, cov_own, out)
        cfg = {"workload": w.name, "order": w.order, "rows": H, "width": w.width, "strip_rows": y1 - y0,
               "halo_rows": g.halo, "super_tile": g.super_tile,
               "parallelism": "row strips over %d ranks, halo exchange by ncclSend/ncclRecv in the library" % world}
        scaling = "strong"
    for _ in range(args.warmup):  # W >= 3 (config 5: minutes per step on few GPUs)
        step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(args.steps):
        step()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / args.steps
    t = torch.tensor([ms, float(npx_rank)], dtype=torch.float64, device=dev)
    if dist:
        dist.all_reduce(t[:1], op=dist.ReduceOp.MAX)
        dist.all_reduce(t[1:], op=dist.ReduceOp.SUM)
    ms, npx = float(t[0]), float(t[1])
    st = plan.stats(reset=True)
    if rank == 0:
        print(json.dumps({"metric": METRIC, "value": npx / (ms * 1e-3) / 1e6, "unit": UNIT, "n_gpus": world,
                          "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
                          "scaling": scaling, "vs_baseline": None, "dtype": "f32 in, f64 out", "data": "synthetic",
                          "config": cfg, "stats": {k: st[k] for k in ("pixels", "double_double", "macs")}}))
    if dist:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--orders", default="", help="comma list; default: the config's orders (config 3: 1,2,3,4)")
    ap.add_argument("--impl", default="bsf")
    ap.add_argument("--ref-points", type=int, default=0, help="oracle pixels per reference step (0: ~0.5 s of work)")
    ap.add_argument("--cpu-budget", type=float, default=8.0, help="seconds of oracle time per order")
    ap.add_argument("--r4-tiles", type=int, default=2368, help="order 4: anchoring tiles sampled (16 per SM)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--frames", type=int, default=64, help="config 4: frames in total (BASELINE.json: 64)")
    ap.add_argument("--frames-per-gpu", type=int, default=0, help="config 4: frames per rank (weak scaling)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.config in (4, 5):
        # the partitioned configs: minutes per step on one GPU (order 3); opt-in
        if args.frames_per_gpu:
            args.frames = args.frames_per_gpu * world
        if args.impl == "reference":
            if rank == 0:
                run_reference(args, synth.workload(args.config), [synth.workload(args.config).order])
            return
        run_partitioned(args, rank, world, local)
        return
    w = synth.workload(args.config)
    orders = [int(x) for x in args.orders.split(",")] if args.orders else ([1, 2, 3, 4] if args.config == 3
                                                                          else [w.order])

    if args.impl == "reference":
        if rank == 0:
            run_reference(args, synth.workload(args.config, order=orders[0]), orders)
        return

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
        pg = dist
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)  # 256 MB > L2
    stream = torch.cuda.current_stream()
    res = {}
    with ClockSampler(local) as clk:
        for r in orders:
            res[r] = time_order(args, synth.workload(args.config, order=r), r, dev, rank, world, stream, flush, pg)
            torch.cuda.empty_cache()
    if rank != 0:
        if pg:
            pg.destroy_process_group()
        return
    if not args.no_cpu_baseline:
        for r in orders:
            res[r]["cpu_baseline"] = cpu_baseline(synth.workload(args.config, order=r), r, args.cpu_budget,
                                                  {1: 50000, 2: 4000}.get(r, 400))
    h = orders[0]
    hw = synth.workload(args.config, order=h)
    line = {"metric": METRIC, "value": res[h]["value"], "unit": UNIT, "n_gpus": world, "steps": res[h]["steps"],
            "warmup": res[h]["warmup"], "ms_per_step": res[h]["ms_per_step"], "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u8 in, int64 sums, f64 out" if hw.in_dtype == "u8"
            else "f32 in, f64", "data": "synthetic",
            "config": {"workload": hw.name, "order": h, "orders": orders, "width": hw.width, "height": hw.height,
                       "basis": "dual" if hw.basis == 2 else str(hw.basis), "in_dtype": hw.in_dtype,
                       "mode": res[h]["mode"], "l2": "flushed between steps (256 MB write, untimed)",
                       "parallelism": "dp%d (independent frames)" % world},
            "roofline": res[h]["roofline"], "cpu_baseline": res[h].get("cpu_baseline"), "e2e": res[h]["e2e"],
            "gpu_launches": res[h]["gpu_launches"], "clocks": clk.summary(), "stats": res[h]["stats"],
            "orders": {str(r): res[r] for r in orders}}
    print(json.dumps(line))
    if pg:
        pg.destroy_process_group()


if __name__ == "__main__":
    main()
