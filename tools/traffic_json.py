"""Write profiles/r02_traffic.json (DRAM bytes per launch, keyed by the hash of
the CUDA sources the captures were taken on) from ncu --set full raw CSV
exports: dram__bytes_read.sum + dram__bytes_write.sum per kernel family.

python tools/traffic_json.py  (after tools/gpu/r02_final2.sh's r02_r1_full_raw.csv /
r02_r{2,3}_fused_raw.csv exports were copied into profiles/)."""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import _src_hash  # noqa: E402

UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def per_kernel(path):
    rows = list(csv.reader(open(os.path.join(ROOT, path))))
    h, units = rows[0], rows[1]
    ik, ir, iw = h.index("Kernel Name"), h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
    out = []
    for r in rows[2:]:
        b = float(r[ir]) * UNIT[units[ir]] + float(r[iw]) * UNIT[units[iw]]
        out.append((r[ik], b))
    return out


def main():
    sh = _src_hash()
    caps = {}
    r1 = per_kernel("profiles/r02_r1_full_raw.csv")
    scans = [b for k, b in r1 if "scan_" in k]
    gx = [b for k, b in r1 if "gx1_kernel" in k]
    caps["c3_4096_u8_grid32/r1/scan"] = {"dram_bytes": sum(scans), "src_hash": sh, "launches": len(scans),
                                         "file": "profiles/r02_r1_full_raw.csv"}
    caps["c3_4096_u8_grid32/r1/gx1_kernel"] = {"dram_bytes": gx[0], "src_hash": sh,
                                               "file": "profiles/r02_r1_full_raw.csv"}
    for r in (2, 3):
        path = "profiles/r02_r%d_fused_raw.csv" % r
        if os.path.exists(os.path.join(ROOT, path)):
            rr = per_kernel(path)
            caps["c3_4096_u8_grid32/r%d/fused_kernel" % r] = {"dram_bytes": rr[0][1], "src_hash": sh, "file": path}
    path = "profiles/r02_r4_tile_raw.csv"
    if os.path.exists(os.path.join(ROOT, path)):
        rr = [b for k, b in per_kernel(path) if "tile_kernel" in k]
        caps["c3_4096_u8_grid32/r4/tile_kernel"] = {"dram_bytes": rr[0], "src_hash": sh, "file": path}
    # order 4: the 10.5 s launch did not finish an ncu --set full capture within
    # 20 min (tools/gpu/r02_close.sh); its DRAM bytes come from the metrics pass
    # of the same launch (long-format CSV: one row per metric)
    path = "profiles/r02_r4_launches.csv"
    key = "c3_4096_u8_grid32/r4/tile_kernel"
    if key not in caps and os.path.exists(os.path.join(ROOT, path)):
        rows = [r for r in csv.reader(open(os.path.join(ROOT, path))) if len(r) > 14 and "tile_kernel" in r[4]]
        b = sum(float(r[14]) * UNIT[r[13]] for r in rows if r[0] == rows[0][0] and r[12].startswith("dram__bytes_"))
        caps[key] = {"dram_bytes": b, "src_hash": sh, "file": path,
                     "capture": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum (not --set full)"}
    doc = {"what": "dram__bytes_read.sum + dram__bytes_write.sum per launch (per step for the 8 scan launches of "
                   "order 1), one ncu --set full --clock-control none capture of tools/step_probe.py on config 3 "
                   "(tools/gpu/r02_final2.sh); bench.py reports them only while src_hash matches the CUDA sources",
           "src_hash": sh, "captures": caps}
    with open(os.path.join(ROOT, "profiles", "r02_traffic.json"), "w") as fh:
        json.dump(doc, fh, indent=1)
    print(json.dumps(doc, indent=1))


if __name__ == "__main__":
    main()
