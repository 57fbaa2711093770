# Round-end evidence bundle: config-2 bench + ncu launch list + traffic + fc1-wgrad full capture,
# ResNet-8 (config 5) launch list, and the per-config sweep.
bash tools/profile_round.sh
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file gpurun_out/resnet_launches.csv python tools/resnet_probe.py > /dev/null 2>&1
python tools/summarize_launches.py gpurun_out/resnet_launches.csv > gpurun_out/resnet_launches_summary.txt
timeout 600 python tools/config_sweep.py > gpurun_out/config_sweep_final.jsonl 2> gpurun_out/config_sweep_final.err
python tools/resnet_probe.py > gpurun_out/resnet_probe.json
cat gpurun_out/traffic.txt gpurun_out/launches_summary.txt gpurun_out/resnet_launches_summary.txt gpurun_out/resnet_probe.json
