mkdir -p gpurun_out/r02z5
O=gpurun_out/r02z5
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off -k regex:k_jacobi_cluster --csv --log-file $O/jc_times.csv python scripts/traffic.py run C4 4096 20 > $O/ncu1.log 2>&1
IDX=$(python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/r02z5/jc_times.csv')))
hi=[i for i,r in enumerate(rows) if 'Metric Value' in r][0]
h=rows[hi]; vi=h.index('Metric Value'); ui=h.index('Metric Unit')
best=(0,-1)
for n,r in enumerate(rows[hi+1:]):
    if len(r)<=vi: continue
    v=float(r[vi].replace(',',''))*{'nsecond':1e-3,'usecond':1,'msecond':1e3}.get(r[ui],1)
    if v>best[0]: best=(v,n)
print(best[1])
PY
)
echo "longest k_jacobi_cluster launch index $IDX" > $O/idx.txt
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:k_jacobi_cluster -s $IDX -c 1 -f -o $O/k_jacobi_cluster python scripts/traffic.py run C4 4096 20 > $O/ncu2.log 2>&1
cat $O/idx.txt; tail -2 $O/ncu2.log
