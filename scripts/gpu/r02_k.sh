cd $GRAFT_REPO_ROOT
for lib in paper_2406_17808_b200/libcascade.so build/lib_se5.so build/lib_se6.so build/lib_se8.so build/lib_fe2.so build/lib_fe6.so; do
  echo "== $lib"; CASCADE_LIB=$lib timeout 120 python scripts/kbench.py 200 6 2>&1 | grep -E "attn_|total"
done
for lib in paper_2406_17808_b200/libcascade.so build/lib_se6.so build/lib_se8.so; do
  echo "== bench $lib"; CASCADE_LIB=$lib timeout 600 python bench.py --steps 3 --warmup 3 --no-decode --no-e2e --no-cpu --no-onepass 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), d['kernels']['attn_fwd']['ms_per_step'], d['kernels']['attn_score']['ms_per_step'], d['clocks']['sm_mhz'])"
done
