# Round-2 final evidence (final code): GPU suite, smoke(), bench lines (driver command; config 5 strong),
# ncu launch list + traffic + fc1-wgrad capture, config-2 per-kernel ncu table, per-config sweep.
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/final_pytest.log 2>&1; echo "pytest rc=$?"
tail -n 2 gpurun_out/final_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo "smoke rc=$?"; tail -n 5 gpurun_out/final_smoke.log
timeout 300 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/final_bench_c2.json 2> gpurun_out/final_bench_c2.err; echo "bench c2 rc=$?"
timeout 300 python bench.py --config 5 --scaling strong --steps 20 --warmup 5 > gpurun_out/final_bench_c5.json 2> gpurun_out/final_bench_c5.err; echo "bench c5 rc=$?"
cut -c1-300 gpurun_out/final_bench_c2.json gpurun_out/final_bench_c5.json
timeout 300 python tools/resnet_probe.py > gpurun_out/final_resnet_probe.json 2>&1
timeout 300 python tools/tail_probe.py > gpurun_out/final_tail.json 2>&1
bash tools/profile_round.sh > gpurun_out/profile_round.log 2>&1; echo "profile_round rc=$?"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed
timeout 1500 ncu --profile-from-start off --metrics $M --clock-control none --csv --log-file gpurun_out/ncu_c2.csv \
  python tools/prof_round.py > gpurun_out/ncu_c2.log 2>&1
python tools/ncu_table.py gpurun_out/ncu_c2.csv > gpurun_out/ncu_table_config2.txt; head -20 gpurun_out/ncu_table_config2.txt
timeout 900 python tools/config_sweep.py > gpurun_out/final_config_sweep.jsonl 2> gpurun_out/final_config_sweep.err; echo "sweep rc=$?"
