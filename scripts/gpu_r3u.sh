O=gpurun_out/final7b; mkdir -p $O
export PATH=/usr/local/cuda/bin:$PATH
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_gemm$" -c 40 -o /tmp/kg python scripts/profile_c5a.py --records $O/recs.json > $O/ncu_kg.log 2>&1; echo "ncu kg exit $?"
ncu -i /tmp/kg.ncu-rep --page raw --csv > /tmp/kg_raw.csv 2>/dev/null
python - <<'PY'
import csv
rows=list(csv.reader(open('/tmp/kg_raw.csv')))
hdr,units,data=rows[0],rows[1],rows[2:]
it=hdr.index('gpu__time_duration.sum')
b=max(data,key=lambda r: float(r[it].replace(',','')))
w=csv.writer(open('gpurun_out/final7b/ncu_full_kgemm_top_launch_raw.csv','w')); w.writerow(hdr); w.writerow(units); w.writerow(b)
print(len(data), b[hdr.index('Kernel Name')], b[it])
PY
