"""Phase breakdown of the fused tile kernel on a BASELINE config (GPU).

python tools/phase_profile.py [--config 2] [--order R]
Prints the share of SM cycles per phase (diagnostic counters, one clock read
per phase per tile; see bsf_debug_phase_cycles)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1109_5114_b200 import bsf  # noqa: E402

PHASES = ["scales (reach)", "preint: zero pads", "exact split (global: setup)", "scatter", "gather", "accumulate"]

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--order", type=int, default=0)
ap.add_argument("--anchor", default="tile", choices=["tile", "global", "auto"])
args = ap.parse_args()
w = synth.workload(args.config, order=args.order) if args.order else synth.workload(args.config)
dev = torch.device("cuda:0")
plan = bsf.Plan(w.width, w.height, in_dtype=bsf.BSF_U8 if w.in_dtype == "u8" else bsf.BSF_F32, order=w.order,
                basis=w.basis, max_sigma=w.max_sigma,
                anchor={"tile": bsf.BSF_ANCHOR_TILE, "global": bsf.BSF_ANCHOR_GLOBAL, "auto": bsf.BSF_ANCHOR_AUTO}[args.anchor])
img = synth.make_image(w, device=dev).contiguous()
cov = synth.make_cov(w, device=dev).contiguous()
out = torch.empty((1, w.height, w.width), dtype=torch.float64, device=dev)
plan.run(img, cov, out)
plan.phase_cycles(reset=True)
plan.stats(reset=True)
plan.run(img, cov, out)
cyc = plan.phase_cycles()
st = plan.stats(reset=True)
print("pixels %d, double-double fallback %d (%.3f %%), macs/px %.0f" % (
    st["pixels"], st["double_double"], 100.0 * st["double_double"] / max(st["pixels"], 1),
    st["macs"] / max(st["pixels"], 1)))
tot = sum(cyc[:6]) + cyc[8] + cyc[9] + cyc[10] + cyc[11] + cyc[12]
print("workload", w.name, "fused", plan.uses_fused())
for n, c in zip(PHASES, cyc):
    print("%-16s %6.1f%%  %.3e cycles" % (n, 100.0 * c / tot, c))
for n, c in (("sub-tile scales", cyc[8]), ("keys", cyc[9]), ("bucket scan", cyc[10]),
             ("  preint: sweeps", cyc[11]), ("  preint: variants", cyc[12])):
    print("%-16s %6.1f%%  %.3e cycles" % (n, 100.0 * c / tot, c))
print("gather groups: warp-cycles total %.3e, full-variant MMA loop %.3e (per-CTA wall equivalent /8: %.3e, %.3e)"
      % (cyc[6], cyc[7], cyc[6] / 8, cyc[7] / 8))
if cyc[15]:
    # executed MMA work per limb (incl. item, window-slot and column padding) vs the algorithmic MACs
    print("MMA padding: item fill %.3f (%d real / %d group slots), executed/algorithmic MACs per limb %.3f"
          % (cyc[14] / cyc[15], cyc[14], cyc[15], cyc[13] / max(st["macs"], 1)))
