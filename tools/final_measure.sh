#!/bin/bash
# Round-end measurement set: bench lines (both arms) for every config, the ncu
# launch list of the default bench command, one full ncu capture of the top
# kernel. Outputs under gpurun_out/final/.
mkdir -p gpurun_out/final
for c in rqc28 hea20 qaoa30 noisy15 rqc33; do
  K=5; [ "$c" = hea20 ] && K=50   # 2 ms steps: a longer timed region
  timeout 900 python bench.py --config $c --steps $K > gpurun_out/final/bench_$c.json 2> gpurun_out/final/bench_$c.err
  timeout 600 python bench.py --impl reference --config $c --steps 2 > gpurun_out/final/ref_$c.json 2> gpurun_out/final/ref_$c.err
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final/launches_rqc28.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/final/ncu_launch.log 2>&1
# three consecutive stage launches of the headline config (after its warm-up steps)
ncu --set full --import-source on --clock-control none -k regex:vqb_stage --launch-skip 70 --launch-count 4 \
    -o gpurun_out/final/ncu_full_rqc28 python bench.py --config rqc28 --no-extra --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/final/ncu_full.log 2>&1
echo done
