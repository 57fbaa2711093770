# Round-end evidence: bench line, ncu launch list (time + DRAM) of the same bench command,
# and one full ncu capture of the dominant kernel in a heavy lock-step iteration.
set -x
timeout 300 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 1 --warmup 1 > gpurun_out/ncu_bench_final.log 2>&1
python tools/ncu_traffic.py gpurun_out/launches_final.csv bf16 profiles/ncu_traffic.json > gpurun_out/traffic.txt
python tools/summarize_launches.py gpurun_out/launches_final.csv > gpurun_out/launches_summary.txt
# dominant kernel (fc1 wgrad: k_gemm_tc launch 2 of each iteration) in heavy lock-step iteration 5
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on \
  -k regex:"k_gemm_tc" --launch-skip 11 --launch-count 1 -o gpurun_out/prof_dom \
  python tools/prof_round.py > gpurun_out/ncu_dom.log 2>&1
# then the bench line again, reading the fresh traffic json
timeout 300 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_final2.json 2> gpurun_out/bench_final2.err
ls -la gpurun_out/launches_final.csv gpurun_out/prof_dom.ncu-rep
