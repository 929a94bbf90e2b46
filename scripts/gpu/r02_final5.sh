cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 900 --timeout-method thread > gpurun_out/pt_final5.log 2>&1; echo pytest rc=$?; grep -E "passed|failed|Error" gpurun_out/pt_final5.log | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
