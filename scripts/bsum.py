"""Summarise bench.py JSON lines: python scripts/bsum.py file..."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads([l for l in open(f).read().splitlines() if l.startswith("{")][-1])
    except Exception as e:  # noqa: BLE001
        print(f, "unreadable", e)
        continue
    st = d.get("stages", {})
    eo = d.get("embedding_only") or {}
    es = eo.get("stage_ms_per_step", {})
    print(f"{f}: ET {d['value']/1e6:.2f}M {d['ms_per_step']:.3f}ms frac {d['roofline']['frac']:.3f} "
          f"({d['roofline']['kernel']}) | pool {st.get('pool',{}).get('ms_per_step',0):.3f} "
          f"segsum {st.get('segsum',{}).get('ms_per_step',0):.3f} | E {eo.get('ms_per_step',0):.3f}ms "
          f"frac {eo.get('roofline',{}).get('frac',0):.3f} pool {es.get('pool',0):.3f} seg {es.get('segsum',0):.3f} "
          f"sort {es.get('sort',0):.3f} route {es.get('route',0):.3f} | clk {(d.get('clocks') or {}).get('sm_mhz')}")
    zc = d.get("zero_copy")
    if zc:
        print(f"    zero-copy: ET {zc['et']['samples_per_s']/1e6:.2f}M {zc['et']['ms_per_step']:.3f}ms "
              f"frac {zc['et']['roofline']['frac']:.3f} | E {zc['e']['ms_per_step']:.3f}ms "
              f"frac {zc['e']['roofline']['frac']:.3f} whole {zc['e']['whole_step_hbm']['frac']:.3f}")
