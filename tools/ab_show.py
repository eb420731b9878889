#!/usr/bin/env python
"""Summarise tools/stage_breakdown.py JSON lines: per run, the graph V-cycle time and the
per-stage totals (µs per cycle) and per-level ghost/smooth/restrict times."""
import json
import sys

for l in open(sys.argv[1]):
    d = json.loads(l)
    if "graph_ms_per_vcycle" in d:
        print(f"{d['cfg']:6s} lib={d.get('lib') or 'tree'} extra={d.get('extra')} "
              f"V-cycle {d['graph_ms_per_vcycle']:.4f} ms  runs={[round(x, 3) for x in d.get('runs', [])]}")
    else:
        r = d["us_per_cycle[stage][level]=(us, launches)"]
        tot = {k: round(sum(v[0] for v in vv.values()), 1) for k, vv in r.items()}
        print("   ", tot)
        for st in sys.argv[2:]:
            if st in r:
                print("      ", st, {m: v[0] for m, v in r[st].items()})
