set -x
free -g; nproc; lscpu | head -20; which numactl; numactl --hardware 2>&1 | head; nvidia-smi -L; df -h /tmp | tail -1
python -c "import __graft_entry__ as g; g.build()" 
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 300 python bench.py > gpurun_out/r2_bench0.json 2> gpurun_out/r2_bench0.err; tail -3 gpurun_out/r2_bench0.err
