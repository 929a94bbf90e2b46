cd $GRAFT_REPO_ROOT
timeout 120 python scripts/kbench.py 200 6 4096 onepass 2>&1 | grep -E "ms/chunk|total"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_fwd_tc -s 2 -c 1 -o gpurun_out/prof_fwd_est python scripts/kbench.py 200 3 4096 onepass > gpurun_out/ncu_fwd_est.log 2>&1; echo ncu rc=$?
