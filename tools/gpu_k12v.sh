mkdir -p gpurun_out
for v in "" "CR_K12_SPLIT=1" "CR_K12_OLD=1"; do
  env $v timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_births|k_apparent|k_codes|k_tags" --csv --log-file gpurun_out/k12v.csv python tools/k12_once.py c5 > /dev/null 2>&1
  echo "variant [$v]"
  python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/k12v.csv')))
hdr=None; d={}
for r in rows:
    if 'Kernel Name' in r: hdr=r; continue
    if hdr and len(r)==len(hdr):
        x=dict(zip(hdr,r)); k=(x['ID'], x['Kernel Name'].split('::')[-1].split('(')[0]); d.setdefault(k,{})[x['Metric Name']]=float(x['Metric Value'].replace(',',''))
for (i,k),m in sorted(d.items(), key=lambda t:int(t[0][0]))[-3:]:
    print(' ',k, round(m['gpu__time_duration.sum']/1000,3),'ms', round((m['dram__bytes_read.sum']+m['dram__bytes_write.sum'])/1e9,3),'GB')
PY
done
