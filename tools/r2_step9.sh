mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s9_build.txt 2>&1 || { tail -30 gpurun_out/s9_build.txt; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_contracts.py tests/test_gpu_autodiff.py -q -x > gpurun_out/s9_tests.txt 2>&1
tail -5 gpurun_out/s9_tests.txt
for c in qaoa30 noisy15 hea20 rqc28; do
  timeout 400 python bench.py --config $c --no-cpu-baseline --no-e2e --no-extra --steps 5 > gpurun_out/s9_$c.json 2>gpurun_out/s9.err
  echo "$c $(python -c "import json;d=json.load(open('gpurun_out/s9_$c.json'));r=d['roofline'];print(round(d['value'],4), round(d['ms_per_step'],3), round(r['frac'],3), round(r.get('fp64',{}).get('frac',0),3), r['launches_per_step'], d['clocks']['sm_mhz'])")" | tee -a gpurun_out/s9_ab.txt
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:vqb_rev -s 30 -c 1 -o gpurun_out/s9_qaoa_rev python bench.py --config qaoa30 --no-extra --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/s9_ncu_qaoa.log 2>&1; echo "ncu qaoa rc=$?"
