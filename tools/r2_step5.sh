# config-4 reference golden on the host cores (background) while the GPU runs
# compute-sanitizer and adjoint ncu captures
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s5_build.txt 2>&1 || { tail -30 gpurun_out/s5_build.txt; exit 1; }
cp tests/golden/fullsize.json gpurun_out/fullsize4.json
( python tests/golden/make_fullsize_golden.py gpurun_out/fullsize4.json config4 > gpurun_out/fullsize4.log 2>&1 ) &
GOLD=$!
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s5_smoke.txt 2>&1; tail -2 gpurun_out/s5_smoke.txt
bash tools/sanitize.sh
timeout 900 ncu --set full --clock-control none --import-source on -k regex:vqb_rev -s 30 -c 1 -o gpurun_out/s5_qaoa_rev python bench.py --config qaoa30 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/s5_ncu_qaoa.log 2>&1; echo "ncu qaoa rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:vqb_rev -s 40 -c 1 -o gpurun_out/s5_noisy_rev python bench.py --config noisy15 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/s5_ncu_noisy.log 2>&1; echo "ncu noisy rc=$?"
wait $GOLD; echo "golden rc=$?"; tail -3 gpurun_out/fullsize4.log
