set -x
timeout 300 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"k_conv2_wgrad_halo|k_conv1_wgrad_q" --launch-skip 10 --launch-count 2 -o gpurun_out/p_heavy python tools/prof_round.py > gpurun_out/p_heavy.log 2>&1
timeout 300 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"k_conv2_wgrad_halo|k_conv1_wgrad_q|k_stage_x|k_head_cnn|QuadConv1" --launch-skip 200 --launch-count 5 -o gpurun_out/p_tail python tools/prof_round.py tail > gpurun_out/p_tail.log 2>&1
PROTEA_DBG=1 python paper_2207_01053_b200/build.py > /dev/null && timeout 200 python tools/dbg_counters.py > gpurun_out/dbg.txt 2>&1
cat gpurun_out/dbg.txt
