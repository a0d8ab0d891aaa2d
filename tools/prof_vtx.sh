#!/bin/bash
# ncu capture of the V^T x kernel of the propagator step (after coarsening) + plan verbose log
OUT=gpurun_out
LEVYH_PLAN_VERBOSE=1 timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu > $OUT/vtx_bench.json 2> $OUT/vtx_bench.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"vtx_kernel|seg_tma_kernel|treduce" \
    -s 12 -c 3 -o $OUT/vtx_prof python bench.py --steps 2 --warmup 3 --no-cpu > $OUT/ncu_vtx.log 2>&1
echo "ncu rc=$?"
