cd $GRAFT_REPO_ROOT
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_r02_v3.json 2> gpurun_out/bench_r02_v3.err; echo bench_rc=$?
python -c "
import json;d=json.load(open('gpurun_out/bench_r02_v3.json'))
print('value',d['value'],'e2e',d['e2e']['value'],'fwd',d['roofline']['frac'],'att',d['roofline_other']['attention_total']['frac_of_burst'],'maint',d['roofline_other']['maintenance']['frac'],'share',d['kernel_share'],'dec',d['decode']['value'],d['decode']['hbm_frac'],'clk',d['clocks'],'cpu',d['cpu_baseline']['value'])"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_r02_reference.json 2> gpurun_out/bench_r02_reference.err; echo ref_rc=$?; cut -c1-300 gpurun_out/bench_r02_reference.json
timeout 300 ncu --set full --clock-control none --import-source on -k regex:decode_fused -s 5 -c 1 -o gpurun_out/prof_decode_v2 python scripts/dbench.py 64 8 > gpurun_out/ncu_decode_v2.log 2>&1; echo ncu decode rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
