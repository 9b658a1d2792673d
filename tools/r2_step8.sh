mkdir -p gpurun_out/dump
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s8_build.txt 2>&1 || { tail -30 gpurun_out/s8_build.txt; exit 1; }
timeout 600 python bench.py --config rqc33 --sharded --no-extra --no-cpu-baseline --steps 3 > gpurun_out/s8_sharded_rqc33.json 2> gpurun_out/s8_sharded_rqc33.err; echo "sharded rqc33 rc=$?"; tail -2 gpurun_out/s8_sharded_rqc33.err
timeout 600 python bench.py --config qaoa30 --sharded --no-extra --no-cpu-baseline --steps 3 > gpurun_out/s8_sharded_qaoa30.json 2> gpurun_out/s8_sharded_qaoa30.err; echo "sharded qaoa30 rc=$?"; tail -2 gpurun_out/s8_sharded_qaoa30.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/s8_ref.json 2> gpurun_out/s8_ref.err; echo "ref rc=$?"; tail -2 gpurun_out/s8_ref.err
VQB_JIT_DUMP=gpurun_out/dump timeout 300 python bench.py --config qaoa30 --no-extra --no-cpu-baseline --no-e2e --steps 1 --warmup 3 > /dev/null 2>&1; ls gpurun_out/dump | wc -l
