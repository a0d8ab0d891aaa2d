# H2 step check: CN parity tests, bench (verbose plan log), short launch list of the step kernels
export LEVYH_PLAN_VERBOSE=1
timeout 900 python -m pytest tests/test_gpu_lu.py tests/test_gpu_step_host.py tests/test_gpu_fullsize.py -q -m gpu -x > gpurun_out/h2_tests.log 2>&1; tail -3 gpurun_out/h2_tests.log
grep -h "H2" gpurun_out/h2_tests.log | head -5
timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu > gpurun_out/b_h2.json 2> gpurun_out/b_h2.err; grep -h "H2\|shared" gpurun_out/b_h2.err | tail -4
python -c "
import json; d=json.load(open('gpurun_out/b_h2.json')); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['gpu_launches_per_step'], d['roofline']['per_kernel'])"
unset LEVYH_PLAN_VERBOSE
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"seg_tma|h2_|tgather|vtx" -c 60 --csv --log-file gpurun_out/lh2.csv python bench.py --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/lh2.csv')))
hi=[i for i,r in enumerate(rows) if r and r[0]=='ID'][0]; h=rows[hi]
ki,mi,vi=h.index('Kernel Name'),h.index('Metric Name'),h.index('Metric Value')
for r in rows[hi+1:][-14:]:
    if len(r)>vi: print(r[ki][:50], r[vi])
PY
