"""Text timeline of a bench.py --trace file: per step, every stage interval
(ms from the step's first record), grouped by stream kind."""
import json
import sys

d = json.load(open(sys.argv[1]))
recs = sorted(d["records"], key=lambda r: r[2])
nsteps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
# step boundaries: each "pool" record on compute starts a window
starts = [r[2] for r in recs if r[0] == "pool"]
for k in range(min(nsteps, len(starts) - 1)):
    t0, t1 = starts[k + 1], starts[k + 2] if k + 2 < len(starts) else starts[k + 1] + 10
    print(f"--- step window {k}: {t1 - t0:.3f} ms")
    for r in recs:
        if r[3] >= t0 and r[2] < t1:
            a, b = max(r[2], t0) - t0, min(r[3], t1) - t0
            print(f"  {r[1]:8s} {r[0]:12s} {r[2]-t0:7.3f} -> {r[3]-t0:7.3f}  ({r[3]-r[2]:.3f})")
