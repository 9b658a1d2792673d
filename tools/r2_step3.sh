mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s3_build.txt 2>&1 || { tail -30 gpurun_out/s3_build.txt; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_contracts.py tests/test_gpu_integration.py tests/test_gpu_sharded_cpp.py "tests/test_gpu_parity_fullsize.py::test_qaoa_gradient_default_path" -q > gpurun_out/s3_tests.txt 2>&1
tail -15 gpurun_out/s3_tests.txt
timeout 900 python bench.py > gpurun_out/s3_bench.json 2> gpurun_out/s3_bench.err; echo "bench rc=$?"; tail -3 gpurun_out/s3_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/s3_launches_rqc28.csv python bench.py --config rqc28 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/s3_ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:vqb_stage -s 40 -c 2 -o gpurun_out/s3_rqc28_stage python bench.py --config rqc28 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/s3_ncu_full.log 2>&1; echo "ncu full rc=$?"
