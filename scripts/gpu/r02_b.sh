cd $GRAFT_REPO_ROOT
# round 2 call B: multi-GPU shapes on one GPU, cfg5 at W=1, the NCCL path under torchrun, the
timeout 600 python -m pytest tests/test_gpu_stack.py -m gpu -q -x -s --timeout 500 --timeout-method thread > gpurun_out/pt_stack.log 2>&1; echo stack rc=$?; grep -E "passed|failed|stack:|Error" gpurun_out/pt_stack.log | tail -4
# coupled stack, compute-sanitizer

for w in 2 4 8; do
  timeout 600 python bench.py --shard-of $w --steps 3 --warmup 3 --no-decode --no-e2e --no-cpu > gpurun_out/shard${w}_cfg3.json 2> gpurun_out/shard${w}_cfg3.err; echo shard$w rc=$?
done
timeout 900 python bench.py --workload cfg5 --shard-of 8 --steps 2 --warmup 3 --no-decode --no-e2e --no-cpu > gpurun_out/shard8_cfg5.json 2> gpurun_out/shard8_cfg5.err; echo shard8_cfg5 rc=$?
timeout 900 python bench.py --workload cfg5 --shard-of 8 --streams 1 --steps 2 --warmup 3 --no-decode --no-e2e --no-cpu > gpurun_out/shard8_cfg5_s1.json 2> gpurun_out/shard8_cfg5_s1.err; echo shard8_cfg5_s1 rc=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/torchrun1.json 2> gpurun_out/torchrun1.err; echo torchrun rc=$?
timeout 900 python bench.py --workload stack --layers 4 --steps 2 --warmup 3 > gpurun_out/stack4.json 2> gpurun_out/stack4.err; echo stack4 rc=$?
timeout 1500 python bench.py --workload cfg5 --steps 1 --warmup 3 --no-decode --no-e2e --no-cpu > gpurun_out/cfg5_w1.json 2> gpurun_out/cfg5_w1.err; echo cfg5 rc=$?
for j in shard2_cfg3 shard4_cfg3 shard8_cfg3 shard8_cfg5 shard8_cfg5_s1 torchrun1 stack4 cfg5_w1; do
  python -c "
import json,sys
try:
  d=json.load(open('gpurun_out/$j.json'))
  print('$j', round(d['value']), d.get('ms_per_step'), d['config'].get('heads_per_rank'), d['config'].get('layers'), d.get('kernel_share'), d.get('stack'), (d.get('decode') or {}).get('value'))
except Exception as e: print('$j', 'ERR', e)"
done
for t in memcheck synccheck; do
  timeout 900 compute-sanitizer --tool $t --error-exitcode 9 python scripts/debug/sanitize_run.py gqa 6 > gpurun_out/sanitize_${t}_gqa.log 2>&1; echo $t gqa rc=$?; tail -2 gpurun_out/sanitize_${t}_gqa.log
  timeout 900 compute-sanitizer --tool $t --error-exitcode 9 python scripts/debug/sanitize_run.py toy 8 > gpurun_out/sanitize_${t}_toy.log 2>&1; echo $t toy rc=$?; tail -2 gpurun_out/sanitize_${t}_toy.log
done
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python scripts/debug/sanitize_run.py cfg2 3 > gpurun_out/sanitize_memcheck_cfg2.log 2>&1; echo memcheck cfg2 rc=$?; tail -2 gpurun_out/sanitize_memcheck_cfg2.log
timeout 1200 compute-sanitizer --tool racecheck --error-exitcode 9 python scripts/debug/sanitize_run.py toy 4 > gpurun_out/sanitize_racecheck_toy.log 2>&1; echo racecheck toy rc=$?; tail -2 gpurun_out/sanitize_racecheck_toy.log
timeout 1200 compute-sanitizer --tool racecheck --error-exitcode 9 python scripts/debug/sanitize_run.py gqa 3 > gpurun_out/sanitize_racecheck_gqa.log 2>&1; echo racecheck gqa rc=$?; tail -2 gpurun_out/sanitize_racecheck_gqa.log
