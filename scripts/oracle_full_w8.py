"""SURVEY §8(d) oracle timing: one full W=8 global DLRM step (8 x 65,536
samples, ~27M keys) -- oracle routing over 8 simulated shards + the Eq. 1/2
step, numpy fp64, one thread.  Rows are materialised before the timer
(table creation, not step work).  Prints one JSON line."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import workload as WL  # noqa: E402
from oracle import routing as OR  # noqa: E402
from oracle import step as OS  # noqa: E402


def main():
    cfg = WL.CONFIGS["dlrm"]
    W = 8
    t0 = time.perf_counter()
    batches = [WL.gen_batch(cfg, 0, 0, r) for r in range(W)]
    douts = [WL.gen_dout(0, 0, r, cfg.batch_local * cfg.num_features, cfg.dim, "realistic") for r in range(W)]
    tab = OS.LazyTable(0, cfg.dim)
    tab.get(np.unique(np.concatenate([k for k, _ in batches])))
    t_prep = time.perf_counter() - t0
    t1 = time.perf_counter()
    OR.route_all(batches, W)
    t_route = time.perf_counter() - t1
    OS.sync_step(tab, batches, douts, 1e-3)
    dt = time.perf_counter() - t1
    K = sum(len(k) for k, _ in batches)
    cpu = "unknown"
    for line in open("/proc/cpuinfo"):
        if line.startswith("model name"):
            cpu = line.split(":", 1)[1].strip()
            break
    print(json.dumps({"kind": "oracle", "workload": "dlrm W=8 global step", "samples": W * cfg.batch_local,
                      "keys": K, "seconds": dt, "route_seconds": t_route, "prep_seconds": t_prep,
                      "samples_per_s": W * cfg.batch_local / dt, "cores": 1, "cpu_model": cpu}))


if __name__ == "__main__":
    main()
