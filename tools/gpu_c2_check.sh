cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 -k "tc or teacher or parity or hwm or bigbatch" > gpurun_out/c2_tests.log 2>&1; echo "tests rc=$?"
tail -n 2 gpurun_out/c2_tests.log
timeout 300 python tools/tail_probe.py 2>&1 | cut -c1-500
