"""Per-class DRAM traffic of one GMRES-IR cycle from an ncu launch list.

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --clock-control none --csv --log-file gpurun_out/traffic.csv python tools/profile_cycle.py
    python tools/traffic_from_ncu.py gpurun_out/traffic.csv > profiles/r1_traffic_ir_cycle.json

ncu's default cache control flushes L2 before every launch, so the bytes are
cold-cache DRAM traffic per launch.  The last cycle of the capture (the eager
profiled cycle of tools/profile_cycle.py) is grouped into the kernel classes
bench.py reports; for each class: launches, mean DRAM bytes per launch, mean
ncu duration (serialised, cold: compare shares, not absolutes).
"""

import collections
import csv
import json
import re
import sys

CLASSES = [  # (bench class, kernel-name pattern)
    ("spmv_dot1", r"k_stencil<float, mpg::EpiPlain|k_spmv<float, mpg::EpiPlain|k_csr_warp<float, mpg::EpiPlain"),
    ("dot1", r"k_dot1_wo<float|k_dot1_small<float"),
    ("update_dot", r"k_update_dot_w<float|k_update_dot<float|k_update_dot_small<float"),
    ("update_norm_givens", r"k_update_norm_scale<float|k_update_norm<float"),
    ("step", r"k_step_mega<float"),
]


def main(*paths):
    """Several captures (e.g. the persistent-step and the four-launch cycle) merge by class."""
    merged = {"sources": list(paths), "cache_control": "all (L2 flushed before each launch)", "classes": {}}
    for p in paths:
        merged["classes"].update(_classes(p))
    json.dump(merged, sys.stdout, indent=1)
    print()


def _classes(path):
    rows = list(csv.reader(open(path)))
    hdr, recs = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            recs.append(dict(zip(hdr, r)))
    ks = collections.OrderedDict()
    for d in recs:
        e = ks.setdefault(d["ID"], {"name": d["Kernel Name"]})
        e[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    items = list(ks.values())
    # the last cycle: from the last k_start_ir (IR cycle start) to the end
    starts = [i for i, it in enumerate(items) if "k_start_ir" in it["name"]]
    cyc = items[starts[-1]:] if starts else items
    out = {"classes": {}}
    for cls, pat in CLASSES:
        sel = [it for it in cyc if re.search(pat, it["name"])]
        if not sel:
            continue
        rd = sum(it.get("dram__bytes_read.sum", 0.0) for it in sel)
        wr = sum(it.get("dram__bytes_write.sum", 0.0) for it in sel)
        t = sum(it.get("gpu__time_duration.sum", 0.0) for it in sel)
        out["classes"][cls] = {"launches": len(sel), "dram_bytes_per_launch": (rd + wr) / len(sel),
                               "dram_read_per_launch": rd / len(sel), "dram_write_per_launch": wr / len(sel),
                               "ncu_ns_per_launch": t / len(sel)}
    return out["classes"]


if __name__ == "__main__":
    main(*sys.argv[1:])
