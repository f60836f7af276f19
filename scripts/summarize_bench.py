#!/usr/bin/env python3
"""One-line summary of a bench.py JSON line (used by scripts/variants.sh)."""
import json
import sys

path, tag = sys.argv[1], (sys.argv[2] if len(sys.argv) > 2 else "")
lines = [x for x in open(path) if x.startswith("{")]
if not lines:
    print(tag, "FAILED", open(path).read()[-800:])
    sys.exit(0)
d = json.loads(lines[-1])
r, c = d["roofline"], d["config"]
print(f"{c['paths']:.0e} {tag:22s} {d['value'] / 1e6:8.1f} Mseg/s  ms/step {d['ms_per_step']:8.1f}  "
      f"fwd {r['forward_ms']:7.1f} (K4a {r.get('k_prefix_ms', 0):6.1f})  "
      f"grad {r['gradient_ms']:7.1f} (K5a {r.get('k_path_gradient_ms', 0):6.1f})  "
      f"iter_frac {r['iteration_frac']:.3f}  K4b {r['k_le_forward_ms']:7.1f} K5b {r['k_le_gradient_ms']:7.1f}")
