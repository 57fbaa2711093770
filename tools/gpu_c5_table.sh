# config-5 per-kernel ncu table of the current code + config-2 tail probe (live per-iteration op cost)
cd $GRAFT_REPO_ROOT
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active
timeout 1200 ncu --profile-from-start off --metrics $M --clock-control none --csv --log-file gpurun_out/ncu_c5.csv \
  python tools/resnet_probe.py > gpurun_out/ncu_c5.log 2>&1
python tools/ncu_table.py gpurun_out/ncu_c5.csv > gpurun_out/ncu_table_config5.txt
cat gpurun_out/ncu_table_config5.txt
timeout 300 python tools/tail_probe.py > gpurun_out/tail.json 2>&1
cat gpurun_out/tail.json
