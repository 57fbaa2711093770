# Per-kernel ncu tables (duration, DRAM bytes, tensor pipe, SM throughput, warps active) of one config-2
# round and one config-5 round of the final code (serialised, cold cache); summaries -> gpurun_out/
cd $GRAFT_REPO_ROOT
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active
timeout 1500 ncu --profile-from-start off --metrics $M --clock-control none --csv --log-file gpurun_out/ncu_c2.csv \
  python tools/prof_round.py > gpurun_out/ncu_c2.log 2>&1
python tools/ncu_table.py gpurun_out/ncu_c2.csv > gpurun_out/ncu_table_config2.txt
timeout 1500 ncu --profile-from-start off --metrics $M --clock-control none --csv --log-file gpurun_out/ncu_c5.csv \
  python tools/resnet_probe.py > gpurun_out/ncu_c5.log 2>&1
python tools/ncu_table.py gpurun_out/ncu_c5.csv > gpurun_out/ncu_table_config5.txt
head -20 gpurun_out/ncu_table_config2.txt; head -20 gpurun_out/ncu_table_config5.txt
timeout 900 ncu --profile-from-start off --metrics $M --clock-control none --csv --log-file gpurun_out/ncu_tail.csv \
  python tools/prof_round.py tail > gpurun_out/ncu_tail.log 2>&1
python tools/ncu_table.py gpurun_out/ncu_tail.csv > gpurun_out/ncu_table_config2_tail.txt
head -20 gpurun_out/ncu_table_config2_tail.txt
