#!/bin/bash
# A/B of env-variable variants: tools/ab2.sh "<configs>" "<env1>" "<env2>" ...  (NONE = no variable)
CFGS="$1"; shift
mkdir -p gpurun_out
for round in 1 2; do
for V in "$@"; do
  for C in $CFGS; do
    K=3; [ "$C" = hea20 ] && K=50
    E="$V"; [ "$V" = NONE ] && E="VQB_NOP=1"
    env $E timeout 600 python bench.py --config $C --no-extra --no-e2e --no-cpu-baseline --steps $K --warmup 3 > gpurun_out/ab.json 2>/dev/null
    python - "$C" "$V" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/ab.json").read().strip().splitlines()[-1])
r = d["roofline"]
print(sys.argv[1], sys.argv[2], "value %.4f" % d["value"], "ms %.2f" % d["ms_per_step"], "frac %.3f" % r["frac"],
      {k: round(v["ms"], 1) for k, v in d["kernels"].items() if v["ms"] > 5}, d["clocks"]["sm_mhz"], flush=True)
PY
  done
done
done
