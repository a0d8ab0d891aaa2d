# H2 walk: bench value per subtree split, then the step's launch list at the default split
for sp in 4 5 6 7; do
  LEVYH_H2_SPLIT=$sp timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu > gpurun_out/b_sp$sp.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/b_sp$sp.json')); print('split $sp', d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['per_kernel'])"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"seg_tma|h2_|tgather|vtx" -c 60 --csv --log-file gpurun_out/lh2.csv python bench.py --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/lh2.csv')))
hi=[i for i,r in enumerate(rows) if r and r[0]=='ID'][0]; h=rows[hi]
ki,mi,vi=h.index('Kernel Name'),h.index('Metric Name'),h.index('Metric Value')
for r in rows[hi+1:][-4:]:
    if len(r)>vi: print(r[ki][:50], r[vi])
PY
