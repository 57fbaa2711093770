cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 -k "resnet or config5 or r8 or tc or teacher" > gpurun_out/mixed_tests.log 2>&1; echo "tests rc=$?"
tail -n 2 gpurun_out/mixed_tests.log
timeout 300 python tools/resnet_probe.py 2>&1 | cut -c1-400
timeout 300 python tools/tail_probe.py 2>&1 | cut -c1-500
bash tools/env_sweep.sh
