python bench.py --config c3 --ncols 4096 --nrows 2048 --steps 200 --warmup 10 --no-cpu --no-extra --graph-steps ${GS:-16} 2>&1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c3 ms/step', d['ms_per_step'], 'GCUPS', d['value'], 'tiles', d['config']['active_tiles_last_step'], 'kernel ms', d['roofline']['kernel_ms_per_step'])"
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3_r2.csv python bench.py --config c3 --ncols 4096 --nrows 2048 --steps 16 --warmup 3 --no-cpu --no-extra --roofline-reps 1 > /dev/null 2>&1
python3 - <<'PY'
import csv,collections
rows=list(csv.reader(open('gpurun_out/launches_c3_r2.csv')))
start=[i for i,r in enumerate(rows) if r and r[0]=='ID'][0]; hdr=rows[start]
d=collections.defaultdict(list)
ki=hdr.index('Kernel Name'); vi=hdr.index('Metric Value'); mi=hdr.index('Metric Name')
for r in rows[start+1:]:
    if len(r)>vi and r[mi]=='gpu__time_duration.sum': d[r[ki][:40]].append(float(r[vi].replace(',','')))
for k,v in d.items(): print(f"{k:42s} n={len(v):4d} mean={sum(v)/len(v)/1e3:8.2f}us min={min(v)/1e3:8.2f}")
PY
