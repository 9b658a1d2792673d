mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s10_build.txt 2>&1 || { tail -30 gpurun_out/s10_build.txt; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_contracts.py tests/test_gpu_autodiff.py -q -x > gpurun_out/s10_tests.txt 2>&1
tail -5 gpurun_out/s10_tests.txt
ab() { cfg=$1; shift
  env "$@" timeout 400 python bench.py --config $cfg --no-cpu-baseline --no-e2e --no-extra --steps 5 > gpurun_out/s10_$cfg.json 2>gpurun_out/s10.err
  echo "$cfg $* $(python -c "import json;d=json.load(open('gpurun_out/s10_$cfg.json'));r=d['roofline'];print(round(d['value'],4), round(d['ms_per_step'],3), round(r['frac'],3), round(r.get('fp64',{}).get('frac',0),3), r['launches_per_step'], d['clocks']['sm_mhz'])")" | tee -a gpurun_out/s10_ab.txt
}
ab qaoa30 VQB_JIT_PBANK=1
ab qaoa30 VQB_JIT_PBANK=0
ab noisy15 VQB_JIT_PBANK=1
ab noisy15 VQB_JIT_PBANK=0
ab noisy15 VQB_JIT_REV_BLOCKS=3
ab hea20 VQB_JIT_PBANK=1
ab hea20 VQB_JIT_PBANK=0
ab rqc28 VQB_JIT_PBANK=1
