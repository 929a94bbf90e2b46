cd $GRAFT_REPO_ROOT
for lib in paper_2406_17808_b200/libcascade.so build/lib_lpt.so paper_2406_17808_b200/libcascade.so build/lib_lpt.so; do
  echo "== $lib"; CASCADE_LIB=$lib timeout 120 python scripts/kbench.py 200 8 2>&1 | grep -E "attn_fwd"
done
for lib in paper_2406_17808_b200/libcascade.so build/lib_lpt.so; do
  echo "== bench $lib"; CASCADE_LIB=$lib timeout 600 python bench.py --steps 3 --warmup 3 --no-decode --no-e2e --no-cpu --no-onepass 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), d['kernels']['attn_fwd']['ms_per_step'], d['clocks']['sm_mhz'])"
done
