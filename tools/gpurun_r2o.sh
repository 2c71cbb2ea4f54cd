# c1 latency-mode breakdown: per-launch durations of one compress (serialised by ncu)
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,launch__grid_size --clock-control none -k regex:plz_ --csv \
    --log-file gpurun_out/launches_c1_r2o.csv python tools/probe.py c1 1 > /dev/null 2>&1; echo ncu rc=$?
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/launches_c1_r2o.csv')))
hdr=None
for r in rows:
    if r and r[0]=='ID': hdr=r; continue
    if hdr and len(r)==len(hdr):
        d=dict(zip(hdr,r))
        print(d['ID'], d['Kernel Name'][:60], d['Metric Name'], d['Metric Value'])
PY
