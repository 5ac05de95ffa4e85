"""Benchmark: megapixels/s of (pre-integration + space-variant filter).

python bench.py --gpus N --steps K --warmup W [--config 2] [--anchor tile|global] [--impl reference]

One step = one pass of the whole hot path over the config's synthetic input,
already resident in HBM.  Default (--anchor tile): bsf_run with the running
sums anchored per 32x32 super-tile and the exact split contraction on the FP64
tensor cores, ONE fused kernel.  --anchor global: the paper's
single global pre-integration (bsf_preintegrate) + bsf_filter.  Default
workload: config 2 of BASELINE.json (1024^2 f32, order 2, dual basis).  For
N > 1 (torchrun, one rank per GPU) every rank filters its own image
(independent problems: weak scaling); time = max over ranks.  The L2 (126 MB)
is flushed between timed steps; each step is timed with CUDA events on the
launching stream, flush excluded.

--impl reference times the CPU oracle (the deliberately slow reference arm of
this tier) on bounded pixel samples of the same workload, on rank 0 only.
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


def _ncu_traffic(workload):
    """DRAM bytes per launch of the fused kernel from the committed ncu capture
    of the default workload (None for other workloads)."""
    if workload != "c2_1024_f32_smooth_r2":
        return None
    try:
        import csv
        rows = list(csv.reader(open(os.path.join(ROOT, "profiles", "r01_c2_fused_raw.csv"))))
        d = dict(zip(rows[0], rows[2]))
        unit = dict(zip(rows[0], rows[1]))
        scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        return sum(float(d[k]) * scale[unit[k]] for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    except Exception:
        return None


def _fp64_peak():
    with open(os.path.join(ROOT, "profiles", "r01_fp64_peak.json")) as fh:
        return json.load(fh)


def algorithmic_fma_per_px(order: int, basis_counts) -> float:
    """(r+1)^4 taps x N_r window x (M_r coefficients + 1)
    multiply-adds per pixel, weighted by the basis mix."""
    from paper_1109_5114_b200 import lut
    tot = 0.0
    for b, frac in basis_counts.items():
        v = lut.load(b, order)["variants"][0]
        tot += frac * (order + 1) ** 4 * v["nmax"] * (v["nmon"] + 1)
    return tot


def workload_config(w, world, precision, anchor):
    """The `config` object of the JSON line (shared by both arms)."""
    return {"workload": w.name, "width": w.width, "height": w.height, "order": w.order,
            "basis": "dual" if w.basis == 2 else str(w.basis), "in_dtype": w.in_dtype, "precision": precision,
            "anchor": anchor, "l2": "flushed between steps (256 MB write, untimed)", "parallelism": "dp%d" % world}


def run_reference(args, w):
    """CPU oracle arm: bounded samples of the workload per step."""
    import oracle as O
    img = synth.make_image(w).numpy()
    cov = synth.make_cov(w).numpy()
    per_step = args.ref_points
    nthreads = os.cpu_count() or 1
    pts = synth.sample_points(w, per_step * (args.steps + args.warmup) + 16, seed=11)
    xs, ys = pts[:, 1].numpy(), pts[:, 2].numpy()

    def step(i):
        sl = slice(i * per_step, (i + 1) * per_step)
        O.filter_points(img, xs[sl], ys[sl], cov[0, ys[sl], xs[sl]].astype(np.float64),
                        cov[1, ys[sl], xs[sl]].astype(np.float64), cov[2, ys[sl], xs[sl]].astype(np.float64),
                        policy=w.basis, r=w.order, nthreads=nthreads)

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
            "config": workload_config(w, 1, "oracle: fp64 direct sum with the exact box-spline kernel", "none"),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": nthreads, "kind": "oracle",
                             "sample": "%d stratified pixels per step of %s (direct sum, exact kernel)" % (
                                 per_step, w.name)},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def cpu_baseline(w, budget_s: float, max_points: int):
    """The oracle as it stands, on a bounded sample of the same workload."""
    import oracle as O
    img = synth.make_image(w).numpy()
    cov = synth.make_cov(w).numpy()
    nthreads = os.cpu_count() or 1
    pts = synth.sample_points(w, max_points, seed=12)
    xs, ys = pts[:, 1].numpy(), pts[:, 2].numpy()
    done, t0 = 0, time.perf_counter()
    chunk = max(nthreads, 8)
    while done < max_points and time.perf_counter() - t0 < budget_s:
        sl = slice(done, min(done + chunk, max_points))
        O.filter_points(img, xs[sl], ys[sl], cov[0, ys[sl], xs[sl]].astype(np.float64),
                        cov[1, ys[sl], xs[sl]].astype(np.float64), cov[2, ys[sl], xs[sl]].astype(np.float64),
                        policy=w.basis, r=w.order, nthreads=nthreads)
        done = sl.stop
    dt = time.perf_counter() - t0
    return {"value": done / dt / 1e6, "unit": UNIT, "cores": nthreads, "kind": "oracle",
            "sample": "%d stratified pixels of %s in %.1f s (direct sum with exact box-spline kernel)" % (
                done, w.name, dt)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--order", type=int, default=0)
    ap.add_argument("--impl", default="bsf")
    ap.add_argument("--precision", default="dd", choices=["dd", "fp64", "auto"])
    ap.add_argument("--anchor", default="tile", choices=["global", "tile"])
    ap.add_argument("--ref-points", type=int, default=24)
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    w = synth.workload(args.config)
    if args.order:
        w = synth.workload(args.config, order=args.order)
    if args.config in (4, 5):
        raise SystemExit("configs 4/5 are parity cases; bench times config 2 (or 1/3)")

    if args.impl == "reference":
        if rank == 0:
            run_reference(args, w)
        return

    from paper_1109_5114_b200 import bsf
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
        pg = dist

    prec = {"dd": bsf.BSF_PREC_DD, "fp64": bsf.BSF_PREC_FP64, "auto": bsf.BSF_PREC_AUTO}[args.precision]
    plan = bsf.Plan(w.width, w.height, batch=1, channels=1,
                    in_dtype=bsf.BSF_U8 if w.in_dtype == "u8" else bsf.BSF_F32, out_dtype=bsf.BSF_F64,
                    order=w.order, basis=w.basis, max_sigma=w.max_sigma, precision=prec, device=local,
                    anchor=bsf.BSF_ANCHOR_TILE if args.anchor == "tile" else bsf.BSF_ANCHOR_GLOBAL)
    img = synth.make_image(w, frame=rank, device=dev).contiguous()
    cov = synth.make_cov(w, device=dev).contiguous()
    out = torch.empty((1, w.height, w.width), dtype=torch.float64, device=dev)
    g = plan.empty_g()
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)  # 256 MB > L2
    stream = torch.cuda.current_stream()
    npx = w.width * w.height

    tile = args.anchor == "tile"

    def one_step():
        if tile:
            plan.run(img, cov, out, stream)
            return
        plan.preintegrate(img, g, stream)
        plan.filter(g, cov, out, stream)

    for _ in range(args.warmup):
        one_step()
        flush.zero_()
    torch.cuda.synchronize()
    st = plan.stats(reset=True)

    # --- timed region: K steps, events per step (flush between, untimed) ---
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    mids = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    launches0 = plan.launch_count()
    if pg:
        pg.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            starts[i].record(stream)
            if tile:
                mids[i].record(stream)
                plan.run(img, cov, out, stream)
            else:
                plan.preintegrate(img, g, stream)
                mids[i].record(stream)
                plan.filter(g, cov, out, stream)
            ends[i].record(stream)
            flush.zero_()
        torch.cuda.synchronize()
    if pg:
        pg.barrier()
    launches = plan.launch_count() - launches0
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    pre_ms = [s.elapsed_time(m) for s, m in zip(starts, mids)]
    gat_ms = [m.elapsed_time(e) for m, e in zip(mids, ends)]
    ms = sum(step_ms) / args.steps
    stats = plan.stats(reset=True)
    if pg:
        t = torch.tensor([ms], device=dev)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        ms = float(t[0])
    value = world * npx / (ms * 1e-3) / 1e6

    # --- end to end through the C-ABI with host buffers (pinned) ------------
    f_h = img.cpu().pin_memory()
    c_h = cov.cpu().pin_memory()
    o_h = torch.empty(out.shape, dtype=out.dtype).pin_memory()
    for _ in range(2):
        plan.run_host(f_h, c_h, o_h, stream)
    torch.cuda.synchronize()
    e_s = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    e_e = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    if pg:
        pg.barrier()
    for i in range(args.steps):
        e_s[i].record(stream)
        plan.run_host(f_h, c_h, o_h, stream)
        e_e[i].record(stream)
        flush.zero_()
    torch.cuda.synchronize()
    e2e_ms = sum(a.elapsed_time(b) for a, b in zip(e_s, e_e)) / args.steps
    if pg:
        t = torch.tensor([e2e_ms], device=dev)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        e2e_ms = float(t[0])
    e2e = {"value": world * npx / (e2e_ms * 1e-3) / 1e6, "unit": UNIT,
           "h2d_bytes_per_step": f_h.numel() * f_h.element_size() + c_h.numel() * c_h.element_size(),
           "d2h_bytes_per_step": o_h.numel() * o_h.element_size()}

    if rank != 0:
        if pg:
            pg.destroy_process_group()
        return

    # --- roofline of the dominant kernel ---------------------------------------
    peaks, src = _peaks()
    sm_mhz = peaks.get("sm_max_mhz", 1965.0)
    gh, gw = plan.geometry.g_height, plan.geometry.g_width
    nb = plan.geometry.nbases
    in_b = 1 if w.in_dtype == "u8" else 4
    gat = sum(gat_ms) / len(gat_ms)
    pre = sum(pre_ms) / len(pre_ms)
    if tile and plan.uses_fused():
        # one fused kernel (pre-integration + exact split contraction on the FP64
        # tensor cores); algorithmic work = the interpolation multiply-adds of
        # Eq. (11) the kernel counted (window x monomials per tap, no padding)
        fp = _fp64_peak()
        macs_px = stats["macs"] / max(stats["pixels"], 1)
        achieved = 2.0 * macs_px * npx / (gat * 1e-3) / 1e12
        plan.phase_cycles(reset=True)  # enables the counters (diagnostic pass, untimed)
        plan.run(img, cov, out, stream)
        plan.phase_cycles(reset=True)
        plan.run(img, cov, out, stream)
        c = plan.phase_cycles()  # counters of bsf_debug_phase_cycles (include/bsf.h)
        cyc = [c[0] + c[8], c[1] + c[11] + c[12], c[2], c[3] + c[9] + c[10], c[4], c[5]]
        tot = float(sum(cyc)) or 1.0
        names = ["scales", "pre_integration", "exact_split", "keys_sort", "gather", "accumulate"]
        alg_bytes = npx * in_b + 12 * npx + 8 * npx  # read f + cov once, write out once
        hbm_gbs = alg_bytes / (gat * 1e-3) / 1e9
        roof = {"bound": "tensor", "pipe": "FP64 tensor (DMMA m8n8k4; tcgen05 has no f64 kind)",
                "kernel": "fused_kernel (pre-integration + gather, DMMA m8n8k4)",
                "achieved": achieved, "peak": fp["fp64_tensor_peak_tflops"], "unit": "TFLOP/s",
                "frac": achieved / fp["fp64_tensor_peak_tflops"], "traffic": _ncu_traffic(w.name),
                "hbm": {"algorithmic_bytes": alg_bytes, "achieved_gbs": hbm_gbs, "peak_gbs": peaks.get("hbm_gbs"),
                        "frac": hbm_gbs / peaks.get("hbm_gbs", 6650.0), "peak_source": src},
                "traffic_source": "dram__bytes_read.sum + dram__bytes_write.sum per launch, one ncu --set full "
                                  "capture (profiles/r01_c2_fused_raw.csv); algorithmic HBM bytes %d" % (
                                      npx * in_b + 12 * npx + 8 * npx),
                "peak_source": "measured: tools/fp64_peak.cu DMMA m8n8k4 (profiles/r01_fp64_peak.json)",
                "algorithmic_macs_per_px": macs_px, "executed_limbs": 2, "kernel_ms": gat,
                "share_of_step": gat / ms if ms else None,
                "phase_share": {n: c / tot for n, c in zip(names, cyc)}}
    else:
        fp64_peak = 148 * 64 * 2 * sm_mhz * 1e6 / 1e12  # TFLOP/s: 64 DFMA/clk/SM
        tp = stats["theta_prime"] / max(stats["pixels"], 1)
        fma_px = algorithmic_fma_per_px(w.order, {0: 1 - tp, 1: tp})
        achieved = 2 * fma_px * npx / (gat * 1e-3) / 1e12
        # algorithmic bytes of the pre-integration: read f once, write g (dd) once per basis
        pre_bytes = npx * in_b + nb * gh * gw * 16
        roof = {"bound": "alu", "kernel": "tile_kernel (dd, fused)" if tile else "gather_kernel",
                "achieved": achieved, "peak": fp64_peak, "unit": "TFLOP/s", "frac": achieved / fp64_peak,
                "traffic": None, "peak_source": "148 SM x 64 DFMA/clk x 2 x %.0f MHz (sm_max, %s)" % (sm_mhz, src),
                "algorithmic_fma_per_px": fma_px, "gather_ms": gat,
                "share_of_step": gat / ms if ms else None,
                "preintegration": {"bound": "hbm", "ms": pre, "achieved_gbs": pre_bytes / (pre * 1e-3) / 1e9,
                                   "peak_gbs": peaks.get("hbm_gbs"), "frac": pre_bytes / (pre * 1e-3) / 1e9 /
                                   peaks.get("hbm_gbs", 6650.0), "algorithmic_bytes": pre_bytes}}
    cb = None
    if not args.no_cpu_baseline:
        cb = cpu_baseline(w, args.cpu_budget, 400)
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(
                w, world,
                "exact split contraction (2 fp64 limbs)" if tile and plan.uses_fused() else
                {"dd": "double-double", "fp64": "fp64",
                 "auto": "fp64 + a-posteriori bound, double-double fallback"}[args.precision], args.anchor),
            "roofline": roof, "cpu_baseline": cb, "e2e": e2e, "gpu_launches": launches,
            "clocks": clk.summary(),
            "stats": {k: stats[k] for k in ("pixels", "clamped", "zero_scale", "theta_prime", "flags",
                                            "double_double", "macs")}}
    print(json.dumps(line))
    if pg:
        pg.destroy_process_group()


if __name__ == "__main__":
    main()
