#!/bin/bash
# quick GPU check: gpu tests (subset) + bench lines for the given workloads
# usage: tools/quickbench.sh "<pytest files>" workload...
T="$1"; shift
if [ -n "$T" ]; then python -m pytest $T -m gpu -q -x 2>&1 | tail -1; fi
for C in "$@"; do
  python bench.py --config $C --no-e2e --no-cpu-baseline --steps 5 > gpurun_out/q_$C.json 2>gpurun_out/q_$C.err
  python - "$C" <<'PY'
import json, sys
c = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/q_{c}.json").read().strip().splitlines()[-1])
except Exception as e:
    print(c, "FAILED", open(f"gpurun_out/q_{c}.err").read()[-800:]); sys.exit()
r = d["roofline"]
print(c, round(d["value"], 3), d["unit"], "ms/step %.2f" % d["ms_per_step"], "fp64 %.3f" % r.get("fp64", {}).get("frac", 0),
      "hbm %.3f" % r["frac"], {k: (v["launches"], round(v["ms"], 2)) for k, v in d["kernels"].items()})
PY
done
