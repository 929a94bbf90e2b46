cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
nvidia-smi --query-gpu=timestamp,clocks.sm,power.draw,power.limit,clocks_throttle_reasons.active --format=csv,noheader -lms 100 > gpurun_out/smi_s3k.csv &
SMI=$!
timeout 300 python scripts/kbench.py 200 40 2>&1 | grep -E "attn_fwd|attn_score|total"
CASCADE_LIB=build/lib_noexp.so timeout 300 python scripts/kbench.py 200 40 2>&1 | grep -E "attn_fwd|total"
kill $SMI
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/smi_s3k.csv'))]
busy=[r for r in rows if float(r[2].split()[0])>300]
print(len(rows),'samples;',len(busy),'above 300 W')
for r in busy[::max(1,len(busy)//25)]: print(','.join(x.strip() for x in r))
PY
