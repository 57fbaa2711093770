# Round-2 evidence, part 2: bench lines with the one-instrumented-round timing, config-5 per-kernel ncu
# table of the final code, full captures of the heaviest ResNet halo launches.
cd $GRAFT_REPO_ROOT
timeout 300 python bench.py > gpurun_out/r2_bench_c2.json 2> gpurun_out/r2_bench_c2.err; echo "bench c2 rc=$?"
timeout 300 python bench.py --config 5 --scaling strong > gpurun_out/r2_bench_c5.json 2> gpurun_out/r2_bench_c5.err; echo "bench c5 rc=$?"
cut -c1-300 gpurun_out/r2_bench_c2.json gpurun_out/r2_bench_c5.json
bash tools/gpu_r8_ncu.sh
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed
timeout 1800 ncu --profile-from-start off --metrics $M --clock-control none --csv --log-file gpurun_out/ncu_c5.csv \
  python tools/resnet_probe.py > gpurun_out/ncu_c5.log 2>&1
python tools/ncu_table.py gpurun_out/ncu_c5.csv > gpurun_out/ncu_table_config5.txt
head -30 gpurun_out/ncu_table_config5.txt
