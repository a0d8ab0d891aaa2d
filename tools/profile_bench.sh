#!/bin/bash
# Round profiling recipe (run under gpurun): plain bench with CPU baseline, launch list of the
# bench command, full ncu capture of the dominant step kernel.  Outputs in gpurun_out/.
set -u
OUT=gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,memory.total --format=csv > $OUT/gpu.txt
timeout 1200 python bench.py --steps 100 --warmup 5 > $OUT/bench_plain.json 2> $OUT/bench_plain.err
echo "bench rc=$?"
timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu > $OUT/bench_small.json 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
    --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > $OUT/ncu_launch.log 2>&1
echo "launch list rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"h2s_up_kernel|h2s_down_kernel|xpad_kernel" \
    -s 12 -c 6 -o $OUT/step_prof python bench.py --steps 2 --warmup 3 --no-cpu > $OUT/ncu_full.log 2>&1
echo "full capture rc=$?"
