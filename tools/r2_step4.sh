mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s4_build.txt 2>&1 || { tail -30 gpurun_out/s4_build.txt; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_autodiff.py tests/test_gpu_parity_fullsize.py tests/test_gpu_golden.py tests/test_gpu_fullsize.py -q > gpurun_out/s4_tests.txt 2>&1
tail -15 gpurun_out/s4_tests.txt
ab() { # config, env...
  cfg=$1; shift
  env "$@" timeout 300 python bench.py --config $cfg --no-cpu-baseline --no-e2e --steps 5 > gpurun_out/s4_ab.json 2>gpurun_out/s4_ab.err
  echo "$cfg $* $(python -c "import json;d=json.load(open('gpurun_out/s4_ab.json'));r=d['roofline'];print(round(d['value'],4), round(d['ms_per_step'],3), round(r['frac'],3), round(r.get('fp64',{}).get('frac',0),3), r['launches_per_step'])")" | tee -a gpurun_out/s4_ab.txt
}
ab rqc28 VQB_JIT_FACTOR=1
ab rqc28 VQB_JIT_MODE=persistent
ab rqc28 VQB_JIT_MODE=persistent VQB_JIT_POOL=smem
ab rqc28 VQB_JIT_BLOCKS=3
ab qaoa30 VQB_JIT_FACTOR=1
ab qaoa30 VQB_JIT_FACTOR=0
ab noisy15 VQB_JIT_FACTOR=1
ab noisy15 VQB_JIT_FACTOR=0
ab hea20 VQB_JIT_FACTOR=1
ab hea20 VQB_JIT_FACTOR=0
VQB_HOST_TIMING=1 timeout 300 python bench.py --config hea20 --no-cpu-baseline --no-e2e --steps 5 2> gpurun_out/s4_hea_host_f1.txt >/dev/null
VQB_HOST_TIMING=1 VQB_JIT_FACTOR=0 timeout 300 python bench.py --config hea20 --no-cpu-baseline --no-e2e --steps 5 2> gpurun_out/s4_hea_host_f0.txt >/dev/null
