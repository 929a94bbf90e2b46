cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 900 --timeout-method thread > gpurun_out/pt_final4.log 2>&1; echo pytest rc=$?; grep -E "passed|failed|Error" gpurun_out/pt_final4.log | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_final4.json 2> gpurun_out/bench_final4.err; echo bench_rc=$?
python -c "
import json;d=json.load(open('gpurun_out/bench_final4.json'))
print('value',round(d['value']),'e2e',round(d['e2e']['value']),'onepass',round(d['onepass']['value']),'fwd',round(d['roofline']['frac'],3),'burst',round(d['roofline']['frac_of_burst'],3),'att',round(d['roofline_other']['attention_total']['frac_of_burst'],3),'maint',round(d['roofline_other']['maintenance']['frac'],3),'dec',round(d['decode']['value']),round(d['decode']['hbm_frac'],3),'clk',d['clocks'],'launches',d['gpu_launches'],'cpu',round(d['cpu_baseline']['value'],1))"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 2>/dev/null > gpurun_out/bench_final4_ref.json; cut -c1-200 gpurun_out/bench_final4_ref.json
