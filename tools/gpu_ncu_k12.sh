mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_births|k_apparent|k_codes|k_tags" --csv --log-file gpurun_out/k12_launches.csv python tools/k12_once.py c4 c5 > gpurun_out/k12.log 2>&1; echo ncu=$?
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/k12_launches.csv')))
hdr=None
for r in rows:
    if 'Kernel Name' in r: hdr=r; continue
    if hdr and len(r)==len(hdr):
        d=dict(zip(hdr,r)); print(d['ID'], d['Kernel Name'][:40], d['Metric Name'], d['Metric Value'])
PY
