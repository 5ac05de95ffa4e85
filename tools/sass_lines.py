"""Attribute an ncu source-page SASS export (per-instruction 'Instructions
Executed' and stall samples) to CUDA source lines via nvdisasm's line info.

python tools/sass_lines.py <kernel-mangled-name> <ncu_sass.csv> [cubin] [top]
(the cubin: cuobjdump -xelf all paper_1109_5114_b200/libbsf.so, the kernels
file; built with -lineinfo)."""
import collections
import csv
import re
import subprocess
import sys

kern, csvp = sys.argv[1], sys.argv[2]
cubin = sys.argv[3] if len(sys.argv) > 3 else "/tmp/cub/bsf_kernels.sm_100a.cubin"
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
sass = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
line_of = {}
cur = ("?", 0)
inside = False
for ln in sass.splitlines():
    if ln.startswith("//--------------------- .text."):
        inside = ln.split(".text.")[1].split()[0] == kern
        continue
    if not inside:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
    if m:
        line_of[int(m.group(1), 16)] = (cur, m.group(2).strip())
rows = list(csv.reader(open(csvp)))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hdr]
ia, ie, iw = h.index("Address"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
data = [r for r in rows[hdr + 1:] if len(r) > iw and r[ia].startswith("0x")]
base = int(data[0][ia], 16)
agg = collections.defaultdict(lambda: [0, 0])
ops = collections.defaultdict(lambda: [0, 0])
tot_i = tot_s = 0
for r in data:
    off = int(r[ia], 16) - base
    (src, ins) = line_of.get(off, (("?", 0), "?"))
    ni, ns = int(r[ie] or 0), int(r[iw] or 0)
    agg[src][0] += ni
    agg[src][1] += ns
    ops[ins.split()[0] if ins != "?" else "?"][0] += ni
    tot_i += ni
    tot_s += ns
print("total warp instructions %.3e, stall samples %d" % (tot_i, tot_s))
for src, (ni, ns) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print("%-22s %5d  instr %5.1f%%  samples %5.1f%%" % (src[0], src[1], 100 * ni / tot_i, 100 * ns / max(tot_s, 1)))
print("-- opcodes --")
for op, (ni, _) in sorted(ops.items(), key=lambda kv: -kv[1][0])[:25]:
    print("%-24s %5.1f%%" % (op, 100 * ni / tot_i))
