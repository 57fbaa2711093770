# ncu --set full of the heaviest (iteration 0) launch of the main ResNet-8 halo kernels (config 5 probe round)
cd $GRAFT_REPO_ROOT
run() {
  timeout 600 ncu --profile-from-start off --kernel-name-base demangled -k "regex:$1" --launch-count 1 \
    --set full --import-source on --clock-control none -o gpurun_out/ncu_$2 python tools/resnet_probe.py > gpurun_out/ncu_$2.log 2>&1
  echo "$2 rc=$?"; tail -n 1 gpurun_out/ncu_$2.log
}
run 'RHalo<\(int\)16, \(bool\)1>' rhalo16d
run 'k_r8_wgrad_halo<protea::RWgHalo<\(int\)16>>' wghalo16
run 'RHalo<\(int\)16, \(bool\)0>' rhalo16f
