mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s7_build.txt 2>&1 || { tail -30 gpurun_out/s7_build.txt; exit 1; }
timeout 1800 python -m pytest tests/test_gpu_contracts.py tests/test_gpu_autodiff.py tests/test_gpu_kernels.py tests/test_gpu_parity_fullsize.py -q -x > gpurun_out/s7_tests.txt 2>&1
tail -15 gpurun_out/s7_tests.txt
for c in rqc28 qaoa30 noisy15 rqc33; do
  timeout 400 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 5 > gpurun_out/s7_$c.json 2>gpurun_out/s7.err
  echo "$c $(python -c "import json;d=json.load(open('gpurun_out/s7_$c.json'));r=d['roofline'];print(round(d['value'],4), round(d['ms_per_step'],3), round(r['frac'],3), round(r.get('fp64',{}).get('frac',0),3), r['launches_per_step'])")" | tee -a gpurun_out/s7_ab.txt
done
