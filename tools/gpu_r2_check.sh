cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_tc.py -q -x --timeout 120 -k "halo_passes" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_teacher_forced.py tests/test_gpu_parity.py -q --timeout 300 -k "resnet8 or config5" 2>&1 | tail -3
PROTEA_R8_HALO=7 timeout 120 python tools/resnet_probe.py | cut -c1-400
timeout 600 ncu --profile-from-start off --kernel-name-base demangled -k 'regex:RHalo<\(int\)16, \(bool\)0>' --launch-skip 40 --launch-count 1 --set full --import-source on --clock-control none \
  -o gpurun_out/rhalo16 python tools/resnet_probe.py > gpurun_out/rhalo16.log 2>&1
timeout 600 ncu --profile-from-start off --kernel-name-base demangled -k 'regex:RWgHalo<\(int\)16>' --launch-skip 40 --launch-count 1 --set full --import-source on --clock-control none \
  -o gpurun_out/wghalo16 python tools/resnet_probe.py > gpurun_out/wghalo16.log 2>&1
tail -n 3 gpurun_out/rhalo16.log gpurun_out/wghalo16.log
