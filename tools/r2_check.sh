# GPU tests + one bench line per gradient config (kernel time only), into gpurun_out/$1
D=gpurun_out/${1:-check}; mkdir -p $D
timeout 1500 python -m pytest tests -m gpu -x -q > $D/pytest.txt 2>&1; echo "pytest rc=$?"; tail -5 $D/pytest.txt
for c in ${2:-qaoa30 noisy15 hea20}; do
  K=3; [ "$c" = hea20 ] && K=50
  timeout 600 python bench.py --config $c --no-extra --no-cpu-baseline --no-e2e --steps $K --warmup 3 > $D/bench_$c.json 2> $D/bench_$c.err
  python - $D/bench_$c.json <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
r = d["roofline"]
print(d["config"]["workload"], "value %.4f" % d["value"], "ms %.2f" % d["ms_per_step"], "hbm frac %.3f" % r["frac"], "fp64 %.3f" % r["fp64"]["frac"],
      "bound %.3f" % r["per_launch_bound"]["frac"], {k: round(v["ms"], 1) for k, v in d["kernels"].items() if v["ms"] > 0.5}, d["clocks"]["sm_mhz"])
PY
done
