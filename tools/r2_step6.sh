mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s6_build.txt 2>&1 || { tail -30 gpurun_out/s6_build.txt; exit 1; }
ab() { cfg=$1; shift
  env "$@" timeout 300 python bench.py --config $cfg --no-cpu-baseline --no-e2e --steps 5 > gpurun_out/s6_ab_$cfg.json 2>gpurun_out/s6_ab.err
  echo "$cfg $* $(python -c "import json;d=json.load(open('gpurun_out/s6_ab_$cfg.json'));r=d['roofline'];print(round(d['value'],4), round(d['ms_per_step'],3), round(r['frac'],3), round(r.get('fp64',{}).get('frac',0),3), r['launches_per_step'])")" | tee -a gpurun_out/s6_ab.txt
}
ab rqc28 VQB_JIT_BLOCKS=4
cp gpurun_out/s6_ab_rqc28.json gpurun_out/s6_rqc28_default.json
ab rqc28 VQB_JIT_BLOCKS=5
ab rqc28 VQB_JIT_BLOCKS=6
ab qaoa30 VQB_JIT_REV_BLOCKS=4
ab qaoa30 VQB_JIT_REV_BLOCKS=5
timeout 900 ncu --set full --clock-control none --import-source on -k regex:vqb_stage -s 35 -c 1 -o gpurun_out/s6_rqc28_heavy0 python bench.py --config rqc28 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/s6_ncu0.log 2>&1; echo "ncu0 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:vqb_stage -s 43 -c 1 -o gpurun_out/s6_rqc28_heavy8 python bench.py --config rqc28 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/s6_ncu8.log 2>&1; echo "ncu8 rc=$?"
