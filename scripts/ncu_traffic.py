"""DRAM traffic per stage launch from an `ncu --set full` report.

    python scripts/ncu_traffic.py REPORT.ncu-rep KEY_PREFIX [--out profiles/ncu_traffic.json]

KEY_PREFIX is "<config>/W<world>/N<micro-batches>" of the captured bench
command; bench.py reads `traffic` for its roofline kernel from the resulting
"<KEY_PREFIX>/<stage>" entries.  A stage's traffic is the sum, over the
kernels that make up one launch of the stage, of the average
dram__bytes_read.sum + dram__bytes_write.sum per launch of that kernel.
"""
from __future__ import annotations

import argparse
import collections
import csv
import io
import json
import os
import subprocess

STAGE_KERNELS = {
    "segsum": ("k_segsum_range", "k_segsum_fix", "k_segsum_fix_big",
               "k_seg_heads", "k_segsum_cold", "k_segsum_hot_chunks", "k_segsum_hot_final"),
    "pool": ("k_pool_stream", "k_pool"),
    "gather": ("k_gather",),
    "refresh": ("k_refresh",),
    "update": ("k_reduce_sgd",),
    "send_gather": ("k_send_gather", "k_send_push"),
}


def kernel_rows(rep: str):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"],
                         check=True, capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    ki = hdr.index("Kernel Name")
    cols = {m: hdr.index(m) for m in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum")}
    units = rows[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
             "s": 1.0, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3}
    for r in rows[2:]:
        if len(r) <= max(cols.values()):
            continue
        name = r[ki].split("(")[0].split("<")[0].replace("void ", "").replace("nest::", "").strip()
        vals = {m: float(r[i].replace(",", "")) * scale.get(units[i], 1) for m, i in cols.items()}
        yield name, vals


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("prefix")
    ap.add_argument("--out", default=os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                  "profiles", "ncu_traffic.json"))
    a = ap.parse_args()
    per = collections.defaultdict(list)
    for name, v in kernel_rows(a.report):
        per[name].append(v)
    data = json.load(open(a.out)) if os.path.exists(a.out) else {}
    meta = data.setdefault("_kernels", {})
    for stage, ks in STAGE_KERNELS.items():
        tot, seen = 0.0, []
        for k in ks:
            if k in per:
                n = len(per[k])
                b = sum(x["dram__bytes_read.sum"] + x["dram__bytes_write.sum"] for x in per[k]) / n
                t = sum(x["gpu__time_duration.sum"] for x in per[k]) / n
                tot += b
                seen.append(k)
                meta[f"{a.prefix}/{k}"] = {"launches": n, "dram_bytes_per_launch": b,
                                           "us_per_launch": t * 1e6, "dram_gbs": b / t / 1e9 if t else None}
        if seen:
            data[f"{a.prefix}/{stage}"] = tot
            print(f"{a.prefix}/{stage}: {tot / 1e6:.1f} MB per launch ({', '.join(seen)})")
    json.dump(data, open(a.out, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
