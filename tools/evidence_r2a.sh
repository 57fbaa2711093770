# Round-2 evidence, part 1: bench lines (config 2 default, config 5 strong), ncu launch list + traffic +
# fc1-wgrad capture (profile_round.sh), ResNet-8 probe, compute-sanitizer logs.
cd $GRAFT_REPO_ROOT
timeout 300 python bench.py > gpurun_out/r2_bench_c2.json 2> gpurun_out/r2_bench_c2.err; echo "bench c2 rc=$?"
timeout 300 python bench.py --config 5 --scaling strong > gpurun_out/r2_bench_c5.json 2> gpurun_out/r2_bench_c5.err; echo "bench c5 rc=$?"
timeout 300 python tools/resnet_probe.py > gpurun_out/r2_resnet_probe.json 2>&1
bash tools/profile_round.sh > gpurun_out/profile_round.log 2>&1; echo "profile_round rc=$?"
rm -f gpurun_out/sanitize_rc.txt
bash tools/sanitize_all.sh > gpurun_out/sanitize_all.log 2>&1
cat gpurun_out/sanitize_rc.txt
cut -c1-400 gpurun_out/r2_bench_c2.json gpurun_out/r2_bench_c5.json gpurun_out/bench_final2.json
