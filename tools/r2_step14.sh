mkdir -p gpurun_out/s14
timeout 900 ncu --set full --clock-control none --import-source on -k regex:vqb_rev -s 40 -c 2 -o gpurun_out/s14/noisy_rev python bench.py --config noisy15 --no-extra --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/s14/ncu_noisy.log 2>&1; echo "ncu noisy rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:vqb_rev -s 34 -c 2 -o gpurun_out/s14/qaoa_rev python bench.py --config qaoa30 --no-extra --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/s14/ncu_qaoa.log 2>&1; echo "ncu qaoa rc=$?"
