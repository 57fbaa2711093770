timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file gpurun_out/resnet_launches.csv python tools/resnet_probe.py > /dev/null 2>&1
python tools/summarize_launches.py gpurun_out/resnet_launches.csv > gpurun_out/resnet_launches_summary.txt
python tools/resnet_probe.py > gpurun_out/resnet_probe.json
timeout 600 python tools/config_sweep.py > gpurun_out/config_sweep_final.jsonl 2> gpurun_out/config_sweep_final.err
cat gpurun_out/resnet_probe.json | cut -c1-300
