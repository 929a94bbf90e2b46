# round 2 call A: parity after the prep fast path + stack, bench lines, ncu captures
cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_stack.py -m gpu -q -x -s --timeout 240 --timeout-method thread > gpurun_out/pt_stack.log 2>&1; echo stack rc=$?; grep -E "passed|failed|stack:|Error" gpurun_out/pt_stack.log | tail -4
for f in test_gpu_parity test_gpu_closure test_gpu_api; do
  timeout 1200 python -m pytest tests/$f.py -m gpu -q -x -s --timeout 400 --timeout-method thread > gpurun_out/pt_$f.log 2>&1; echo $f rc=$?; grep -E "passed|failed|Error" gpurun_out/pt_$f.log | tail -3
done
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_r02.json 2> gpurun_out/bench_r02.err; echo bench_rc=$?
python -c "
import json;d=json.load(open('gpurun_out/bench_r02.json'))
print('value',d['value'],'e2e',d['e2e']['value'],'fwd',d['roofline']['frac'],'att',d['roofline_other']['attention_total'],'maint',d['roofline_other']['maintenance']['frac'],'share',d['kernel_share'],'dec',d['decode']['value'],d['decode']['hbm_frac'],'clk',d['clocks'])"
timeout 300 python bench.py --steps 3 --warmup 3 --score-mode onepass --no-decode --no-e2e --no-cpu > gpurun_out/bench_r02_onepass.json 2> gpurun_out/bench_r02_onepass.err; echo bench1p_rc=$?
python -c "
import json;d=json.load(open('gpurun_out/bench_r02_onepass.json'))
print('onepass value',d['value'],'fwd',d['roofline']['frac'],'share',d['kernel_share'])"
# launch list (cold, serialised) over the first chunks of the bench
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"attn_|maint|rope|decode|onepass|ema_|positions" -c 600 --csv --log-file gpurun_out/ncu_launches_r02.csv python bench.py --steps 1 --warmup 3 --no-decode --no-e2e --no-cpu > /dev/null 2>&1; echo ncu_list rc=$?
# full captures at steady state (kbench: cascade filled to ~62K by score injection)
for k in attn_fwd_tc attn_score_tc maint_coop rope_prep; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -o gpurun_out/prof_$k python scripts/kbench.py 200 3 > gpurun_out/ncu_$k.log 2>&1; echo ncu $k rc=$?
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:decode_fused -s 5 -c 1 -o gpurun_out/prof_decode python scripts/dbench.py 64 8 > gpurun_out/ncu_decode.log 2>&1; echo ncu decode rc=$?
ls -la gpurun_out/*.ncu-rep
