#!/bin/bash
# Alternating A/B/... of library builds on one box (dev tool):
#   bash tools/ab_libs.sh ROUNDS "bench args" default lib/variants/x.so ...
# ("default" = lib/libchebykan.so); one JSON line per run in gpurun_out/ab_<tag>_<round>.json
set -u
R=$1; ARGS=$2; shift 2
mkdir -p gpurun_out
for i in $(seq 1 $R); do
  for L in "$@"; do
    tag=$(basename "$L" .so)
    if [ "$L" = default ]; then
      python bench.py --no-cpu-baseline $ARGS > gpurun_out/ab_${tag}_$i.json 2>/dev/null
    else
      CK_LIB_PATH=$L python bench.py --no-cpu-baseline $ARGS > gpurun_out/ab_${tag}_$i.json 2>/dev/null
    fi
  done
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/ab_*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "no result", e); continue
    k = d.get("kernel_ms_per_step", {})
    print(f, f"value {d['value']:.4g} ms/step {d['ms_per_step']:.4f} clk {d['clocks']['sm_mhz'] if d.get('clocks') else None}",
          " ".join(f"{n} {v:.3f}" for n, v in k.items()))
PY
