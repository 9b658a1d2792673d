# lowered stage programs + generated sources of the gradient configs (for tools/jit_inspect.py on the host)
mkdir -p gpurun_out/dump_qaoa30 gpurun_out/dump_noisy15 gpurun_out/dump_hea20
for c in qaoa30 noisy15 hea20; do
  VQB_JIT_DUMP=gpurun_out/dump_$c timeout 600 python bench.py --config $c --no-extra --no-cpu-baseline --no-e2e --steps 2 --warmup 3 > gpurun_out/dump_$c/bench.json 2> gpurun_out/dump_$c/bench.err
  ls gpurun_out/dump_$c | wc -l
done
VQB_HOST_TIMING=1 timeout 300 python tools/host_timing_grad.py hea20 > gpurun_out/host_timing_hea20.txt 2>&1
tail -60 gpurun_out/host_timing_hea20.txt
