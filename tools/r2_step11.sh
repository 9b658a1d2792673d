mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s11_build.txt 2>&1 || { tail -30 gpurun_out/s11_build.txt; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:vqb_rev -s 30 -c 1 -o gpurun_out/s11_qaoa_rev python bench.py --config qaoa30 --no-extra --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/s11_ncu_qaoa.log 2>&1; echo "ncu qaoa rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:vqb_rev -s 40 -c 1 -o gpurun_out/s11_noisy_rev python bench.py --config noisy15 --no-extra --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/s11_ncu_noisy.log 2>&1; echo "ncu noisy rc=$?"
VQB_JIT_DUMP=gpurun_out/dump11 timeout 300 python bench.py --config noisy15 --no-extra --no-cpu-baseline --no-e2e --steps 1 --warmup 3 > /dev/null 2>&1; ls gpurun_out/dump11 | wc -l
