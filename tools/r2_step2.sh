# build, GPU tests (all, no -x), then A/B of the forward emission on config 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s2_build.txt 2>&1 || { tail -30 gpurun_out/s2_build.txt; exit 1; }
timeout 2400 python -m pytest tests -m gpu -q -p no:randomly > gpurun_out/s2_gputests.txt 2>&1
tail -40 gpurun_out/s2_gputests.txt
for v in "VQB_JIT_FACTOR=1" "VQB_JIT_FACTOR=0" "VQB_JIT_FACTOR=1 VQB_REGS=16w"; do
  env $v timeout 300 python bench.py --config rqc28 --no-cpu-baseline --no-e2e --steps 5 > gpurun_out/s2_ab.json 2>gpurun_out/s2_ab.err
  echo "$v $(python -c "import json;d=json.load(open('gpurun_out/s2_ab.json'));print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline'].get('fp64',{}).get('frac'), d['roofline']['launches_per_step'])")" | tee -a gpurun_out/s2_ab.txt
done
