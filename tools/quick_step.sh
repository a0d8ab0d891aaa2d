timeout 900 python -m pytest tests/test_gpu_build.py tests/test_gpu_multirhs.py -q -m gpu -x 2>&1 | tail -2
timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu > gpurun_out/b_v3.json 2> gpurun_out/b_v3.err; tail -2 gpurun_out/b_v3.err
python -c "
import json; d=json.load(open('gpurun_out/b_v3.json')); print(d['value'], d['ms_per_step'], d['gpu_launches_per_step'], d['roofline']['per_kernel'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"seg_tma|rreduce|xpad|tgather" -c 40 --csv --log-file gpurun_out/l3.csv python bench.py --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/l3.csv')))
hi=[i for i,r in enumerate(rows) if r and r[0]=='ID'][0]; h=rows[hi]
ki,mi,vi=h.index('Kernel Name'),h.index('Metric Name'),h.index('Metric Value')
for r in rows[hi+1:][-12:]:
    if len(r)>vi: print(r[ki][:50], r[vi])
PY
