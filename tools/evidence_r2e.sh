# Round-2 final per-kernel ncu tables: config-2 B = 8 tail, config-5 round (final code)
cd $GRAFT_REPO_ROOT
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed
timeout 1200 ncu --profile-from-start off --metrics $M --clock-control none --csv --log-file gpurun_out/ncu_tail.csv \
  python tools/prof_round.py tail > gpurun_out/ncu_tail.log 2>&1
python tools/ncu_table.py gpurun_out/ncu_tail.csv > gpurun_out/ncu_table_config2_tail.txt; head -16 gpurun_out/ncu_table_config2_tail.txt
timeout 1800 ncu --profile-from-start off --metrics $M --clock-control none --csv --log-file gpurun_out/ncu_c5.csv \
  python tools/resnet_probe.py > gpurun_out/ncu_c5.log 2>&1
python tools/ncu_table.py gpurun_out/ncu_c5.csv > gpurun_out/ncu_table_config5.txt; head -30 gpurun_out/ncu_table_config5.txt
