cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests -m gpu -q --timeout 1400 2>&1 | tail -30 > gpurun_out/t_all.log
timeout 900 python tools/global_controls.py 2 > gpurun_out/global_controls.json 2> gpurun_out/global_controls.err
tail -4 gpurun_out/t_all.log; cat gpurun_out/global_controls.json; tail -3 gpurun_out/global_controls.err
