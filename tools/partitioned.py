"""Throughput of the partitioned configs (BASELINE.json configs 4 and 5) on
N GPUs, one process per GPU (torchrun; NCCL for the plumbing):

  torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/partitioned.py --config 4 --frames 8
  torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/partitioned.py --config 5 --rows 4096

config 4: the frames (3 channels each, one covariance field per frame) are
sharded over the ranks (parallel.shard_range), no collective on the data path
(weak in frames per rank if --frames scales with N).  config 5: one image in
super-tile-aligned row strips with the input halo exchange of
parallel.filter_strip (strong scaling; --rows crops the 32768-row image to
bound the run time).  Timing: barrier + synchronize around the timed steps,
CUDA events on the launching stream, max over ranks.  Prints one JSON line
on rank 0 (not a bench.py line: bench times config 2)."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1109_5114_b200 import bsf  # noqa: E402
from paper_1109_5114_b200 import parallel as PL  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, choices=[4, 5], default=4)
ap.add_argument("--frames", type=int, default=4, help="config 4: frames in total (64 in BASELINE.json)")
ap.add_argument("--rows", type=int, default=0, help="config 5: crop to this many rows (0 = all 32768)")
ap.add_argument("--steps", type=int, default=1)
ap.add_argument("--warmup", type=int, default=1)
args = ap.parse_args()

rank = int(os.environ.get("RANK", "0"))
world = int(os.environ.get("WORLD_SIZE", "1"))
local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
dist = None
if world > 1:
    import torch.distributed as dist
    dist.init_process_group("nccl", device_id=dev)

if args.config == 4:
    w = synth.workload(4)
    f0, f1 = PL.shard_range(args.frames, rank, world)
    nf = f1 - f0
    C = w.channels
    plan = bsf.Plan(w.width, w.height, batch=max(nf, 1), channels=C, in_dtype=bsf.BSF_F32, order=w.order,
                    basis=w.basis, max_sigma=w.max_sigma, anchor=bsf.BSF_ANCHOR_TILE, device=local)
    img = torch.stack([synth.make_image(w, frame=f, channel=c, device=dev) for f in range(f0, f1)
                       for c in range(C)]).contiguous() if nf else None
    cov = torch.stack([synth.make_cov(w, frame=f, device=dev) for f in range(f0, f1)]).contiguous() if nf else None
    out = torch.empty((max(nf, 1) * C, w.height, w.width), dtype=torch.float64, device=dev)
    npx_rank = nf * C * w.width * w.height

    def step():
        if nf:
            plan.run(img, cov, out)
    desc = {"workload": w.name, "frames": args.frames, "channels": C, "frames_per_rank": nf,
            "parallelism": "frames sharded over %d ranks" % world}
else:
    w = synth.workload(5)
    H = args.rows or w.height
    tile = 32
    halo = PL.halo_rows(w.max_sigma, w.order, tile)
    st = PL.strip_plan(H, rank, world, halo, tile)
    f_own = synth.make_image(w, window=(st.y0, st.y1, 0, w.width), device=dev).contiguous()
    cov_own = synth.make_cov(w, window=(st.y0, st.y1, 0, w.width), device=dev).contiguous()
    npx_rank = (st.y1 - st.y0) * w.width

    def factory(height):
        p = bsf.Plan(w.width, height, in_dtype=bsf.BSF_F32, order=w.order, basis=w.basis,
                     max_sigma=w.max_sigma, anchor=bsf.BSF_ANCHOR_TILE, device=local, super_tile=tile)
        assert p.geometry.super_tile == tile
        return p

    def step():
        PL.filter_strip(factory, f_own, cov_own, st, H)
    desc = {"workload": w.name, "rows": H, "width": w.width, "strip_rows": st.y1 - st.y0, "halo_rows": halo,
            "parallelism": "row strips over %d ranks, NCCL halo exchange" % world}

for _ in range(args.warmup):
    step()
torch.cuda.synchronize()
if dist:
    dist.barrier()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter()
a.record()
for _ in range(args.steps):
    step()
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / args.steps
wall = (time.perf_counter() - t0) / args.steps
t = torch.tensor([ms, float(npx_rank)], dtype=torch.float64, device=dev)
if dist:
    mx = t.clone()
    dist.all_reduce(mx[:1], op=dist.ReduceOp.MAX)
    tot = t.clone()
    dist.all_reduce(tot[1:], op=dist.ReduceOp.SUM)
    ms, npx = float(mx[0]), float(tot[1])
else:
    npx = float(npx_rank)
if rank == 0:
    print(json.dumps({"metric": "megapixels/sec (pre-integration + space-variant filter)",
                      "value": npx / (ms * 1e-3) / 1e6, "unit": "Mpx/s", "n_gpus": world, "steps": args.steps,
                      "ms_per_step": ms, "wall_s_per_step": wall, "order": w.order, "config": desc}))
if dist:
    dist.destroy_process_group()
