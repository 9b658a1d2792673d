# GPU tests, gradient benches with e2e, host timing of hea20
D=gpurun_out/${1:-check}; mkdir -p $D
timeout 1500 python -m pytest tests -m gpu -x -q > $D/pytest.txt 2>&1; echo "pytest rc=$?"; tail -5 $D/pytest.txt
for c in hea20 qaoa30 noisy15; do
  K=3; [ "$c" = hea20 ] && K=50
  timeout 600 python bench.py --config $c --no-extra --no-cpu-baseline --steps $K --warmup 3 > $D/bench_$c.json 2> $D/bench_$c.err
  python - $D/bench_$c.json <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
r = d["roofline"]
print(d["config"]["workload"], "value %.4f" % d["value"], "ms %.2f" % d["ms_per_step"], "e2e %.4f" % d["e2e"]["value"], "hbm frac %.3f" % r["frac"],
      {k: round(v["ms"], 1) for k, v in d["kernels"].items() if v["ms"] > 0.5}, d["clocks"]["sm_mhz"])
PY
done
VQB_HOST_TIMING=1 timeout 300 python tools/host_timing_grad.py hea20 2>&1 | tail -14
VQB_PLAN_THREADS=0 timeout 300 python bench.py --config hea20 --no-extra --no-cpu-baseline --steps 50 --warmup 3 | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('hea20 serial planning: value %.1f e2e %.1f' % (d['value'], d['e2e']['value']))"
