cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_tc.py -q -x --timeout 120 -k "halo_passes" 2>&1 | tail -15
timeout 600 python -m pytest tests/test_gpu_tc.py tests/test_gpu_teacher_forced.py tests/test_gpu_parity.py -q --timeout 300 -k "resnet8 or config5" 2>&1 | tail -8
for h in 7 1 2 4 0; do echo "mask $h"; PROTEA_R8_HALO=$h timeout 120 python tools/resnet_probe.py | cut -c1-400; done
