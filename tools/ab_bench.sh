#!/bin/bash
# A/B of the default library against a variant build, alternating on one box:
#   bash tools/ab_bench.sh VARIANT.so [rounds] [bench args...]
set -u
V=$1; R=${2:-2}; shift 2 || true
mkdir -p gpurun_out
for i in $(seq 1 $R); do
  python bench.py --no-cpu-baseline "$@" > gpurun_out/ab_A_$i.json 2>/dev/null
  CK_LIB_PATH=$V python bench.py --no-cpu-baseline "$@" > gpurun_out/ab_B_$i.json 2>/dev/null
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/ab_*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "no result", e); continue
    k = d.get("kernel_ms_per_step", {})
    print(f, f"value {d['value']:.0f} ms/step {d['ms_per_step']:.2f} clk {d['clocks']['sm_mhz'] if d.get('clocks') else None}",
          " ".join(f"{n} {k.get(n, 0):.2f}" for n in ("gemm_fwd", "gemm_dx", "gemm_dc")))
PY
