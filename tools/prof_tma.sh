OUT=gpurun_out
timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu > $OUT/b_tma.json 2> $OUT/b_tma.err
LEVYH_SEG_DIRECT=1 timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu > $OUT/b_dir.json 2> $OUT/b_dir.err
for f in b_tma b_dir; do python -c "
import json; d=json.load(open('$OUT/$f.json')); print('$f', d['value'], d['ms_per_step'], d['roofline']['per_kernel'])"; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"seg_tma_kernel|vtx_kernel" -s 6 -c 3 -o $OUT/tma_prof python bench.py --steps 2 --warmup 3 --no-cpu > $OUT/ncu_tma.log 2>&1
echo ncu rc=$?
