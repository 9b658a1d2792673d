#!/bin/bash
# A/B of env-variable variants in one GPU session: tools/ab.sh "<configs>" "<env1>" "<env2>" ...
# prints per-config kernel ms for each variant (2 rounds, alternating)
CFGS="$1"; shift
for round in 1 2; do
for V in "$@"; do
  for C in $CFGS; do
    env $V python bench.py --config $C --no-e2e --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/ab.json 2>/dev/null
    python - "$C" "$V" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/ab.json").read().strip().splitlines()[-1])
print(sys.argv[1], sys.argv[2], "%.2f ms/step" % d["ms_per_step"], {k: round(v["ms"], 1) for k, v in d["kernels"].items() if v["ms"] > 5})
PY
  done
done
done
