#!/bin/bash
# Timing sweep of kernel mappings (no profiler).  Usage: scripts/variants.sh PATHS "variant1" "variant2" ...
P=${1:-1e7}; shift
mkdir -p gpurun_out
for v in "$@"; do
  tag=$(echo "$v" | tr -d ' -')
  timeout 900 python bench.py --paths $P --steps 3 --warmup 3 --no-cpu-baseline --no-e2e $v > gpurun_out/var_${P}_$tag.log 2>&1
  python - "gpurun_out/var_${P}_$tag.log" "$tag" <<'PY'
import json,sys
f,tag=sys.argv[1],sys.argv[2]
l=[x for x in open(f) if x.startswith("{")]
if not l: print(tag, "FAILED", open(f).read()[-800:]); sys.exit()
d=json.loads(l[0]); r=d["roofline"]; c=d["config"]
print(f"{c['paths']:.0e} {tag:22s} {d['value']/1e6:8.1f} Mseg/s  ms/step {d['ms_per_step']:8.1f}  fwd {r['forward_ms']:7.1f}  grad {r['gradient_ms']:7.1f}  iter_frac {r['iteration_frac']:.3f}  trace {c['trace_s']}s sort {c['sort_s']}s")
PY
done
