cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu_parity.py -k "resnet18" -q --timeout 900 2>&1 | tail -30 > gpurun_out/t_r18.log
grep -E "^E  |passed|failed" gpurun_out/t_r18.log | tail -12
