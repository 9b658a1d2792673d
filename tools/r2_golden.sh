# Runs the reference at BASELINE.json's full sizes on the GPU box host (196 GB RAM,
# 16 cores) and writes gpurun_out/fullsize.json (committed as tests/golden/fullsize.json).
mkdir -p gpurun_out
free -g
python tests/golden/make_fullsize_golden.py gpurun_out/fullsize.json config1 config2 config3 config4 2>&1 | tee gpurun_out/fullsize.log
