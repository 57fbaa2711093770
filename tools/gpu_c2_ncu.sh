# ncu --set full of heavy-iteration (iteration 3) launches of conv1 wgrad, fc1 dgrad and conv2 dgrad (config 2)
cd $GRAFT_REPO_ROOT
run() {
  timeout 600 ncu --profile-from-start off --kernel-name-base demangled -k "regex:$1" --launch-skip 3 --launch-count 1 \
    --set full --import-source on --clock-control none -o gpurun_out/ncu_$2 python tools/prof_round.py > gpurun_out/ncu_$2.log 2>&1
  echo "$2 rc=$?"; tail -n 1 gpurun_out/ncu_$2.log
}
run 'k_conv1_wgrad_q' c1w
run 'TmaFc1Dgrad' f1d
run 'HaloConv2Q<\(bool\)1>' c2d
