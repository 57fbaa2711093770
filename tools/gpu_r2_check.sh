cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_tc.py -q -x --timeout 120 -k "halo_passes" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_teacher_forced.py tests/test_gpu_parity.py -q --timeout 300 -k "resnet8 or config5" 2>&1 | tail -3
for h in 7; do echo "mask $h"; PROTEA_R8_HALO=$h timeout 120 python tools/resnet_probe.py | cut -c1-400; done
timeout 600 ncu --profile-from-start off -k regex:RHalo --launch-skip 40 --launch-count 1 --set full --import-source on --clock-control none \
  -o gpurun_out/rhalo16 python tools/resnet_probe.py > gpurun_out/rhalo16.log 2>&1
ncu -i gpurun_out/rhalo16.ncu-rep --page details --csv 2>/dev/null | head -5 | cut -c1-300
