cd $GRAFT_REPO_ROOT
timeout 600 python bench.py --workload cfg2 --steps 20 --warmup 3 --no-e2e --no-cpu --no-decode --no-onepass > gpurun_out/cfg2.json 2> gpurun_out/cfg2.err; echo cfg2 rc=$?
for w in 2 4; do
timeout 1200 python bench.py --workload cfg5 --shard-of $w --steps 1 --warmup 3 --no-decode --no-e2e --no-cpu > gpurun_out/shard${w}_cfg5.json 2> gpurun_out/shard${w}_cfg5.err; echo shard${w}_cfg5 rc=$?
done
timeout 2400 python bench.py --workload stack --layers 32 --steps 1 --warmup 3 > gpurun_out/stack32.json 2> gpurun_out/stack32.err; echo stack32 rc=$?
for j in cfg2 shard2_cfg5 shard4_cfg5 stack32; do
  python -c "
import json
d=json.load(open('gpurun_out/$j.json'))
print('$j', round(d['value']), round(d['ms_per_step'],1), d['config'].get('heads_per_rank'), d['config'].get('layers'), d.get('kernel_share'), d.get('stack'), d.get('roofline',{}).get('frac'))" 2>&1 | tail -1
done
