mkdir -p gpurun_out
timeout 900 python tools/multitenant.py > gpurun_out/mt_p1.json 2> gpurun_out/mt_p1.err
cat gpurun_out/mt_p1.json; tail -3 gpurun_out/mt_p1.err
timeout 300 python tools/prof_ara.py --steps 2 --mode fold > gpurun_out/plainf.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_fold.csv python tools/prof_ara.py --steps 2 --mode fold > gpurun_out/ncu_f.log 2>&1
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/launches_fold.csv')))
hdr=[i for i,r in enumerate(rows) if 'Kernel Name' in r][0]
h=rows[hdr]; ki=h.index('Kernel Name'); vi=h.index('Metric Value'); ui=h.index('Metric Unit')
for r in rows[hdr+1:]:
    if len(r)>vi: print(r[vi], r[ui], r[ki][:70])
PY
