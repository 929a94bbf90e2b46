cd $GRAFT_REPO_ROOT
timeout 120 python scripts/dbench.py 64 64 2>&1 | tail -1
timeout 120 python scripts/dbench.py 64 64 exact 2>&1 | tail -1
timeout 1800 python -m pytest tests -m gpu -q -x --timeout 900 --timeout-method thread > gpurun_out/pt_e.log 2>&1; echo pytest rc=$?; grep -E "passed|failed|Error" gpurun_out/pt_e.log | tail -3
for w in gqa toy; do
timeout 900 compute-sanitizer --tool synccheck --error-exitcode 9 python scripts/debug/sanitize_run.py $w 6 > gpurun_out/sanitize_synccheck_$w.log 2>&1; echo synccheck $w rc=$?; grep -E "ERROR SUMMARY|Device Frame" gpurun_out/sanitize_synccheck_$w.log | sed 's/+0x[0-9a-f]*//' | sort | uniq -c | head -4
done
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_r02_v2.json 2> gpurun_out/bench_r02_v2.err; echo bench_rc=$?
python -c "
import json;d=json.load(open('gpurun_out/bench_r02_v2.json'))
print('value',d['value'],'e2e',d['e2e']['value'],'fwd',d['roofline']['frac'],'traffic',d['roofline']['traffic'],'att',d['roofline_other']['attention_total']['frac_of_burst'],'maint',d['roofline_other']['maintenance']['frac'],'share',d['kernel_share'],'dec',d['decode']['value'],d['decode']['hbm_frac'],'clk',d['clocks'])"
