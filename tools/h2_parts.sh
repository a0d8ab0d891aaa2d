# H2 walk timing experiments (LEVYH_H2_DBG bits skip parts; results are wrong then, timings only)
for d in 0 1 2 4 8; do
  LEVYH_H2_DBG=$d timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"h2_" -c 40 --csv --log-file gpurun_out/lp$d.csv python bench.py --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1
  python - $d <<'PY'
import csv,sys
rows=list(csv.reader(open(f'gpurun_out/lp{sys.argv[1]}.csv')))
hi=[i for i,r in enumerate(rows) if r and r[0]=='ID'][0]; h=rows[hi]
ki,vi=h.index('Kernel Name'),h.index('Metric Value')
print('dbg',sys.argv[1],[(r[ki].split('(')[0].split('::')[-1],r[vi]) for r in rows[hi+1:][-4:] if len(r)>vi])
PY
done
