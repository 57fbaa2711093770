# Round-2 final evidence: GPU suite, bench lines (driver's command), ncu launch list + traffic + fc1-wgrad
# capture, per-config sweep, ResNet probe.
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/final_pytest.log 2>&1; echo "pytest rc=$?"
tail -n 2 gpurun_out/final_pytest.log
timeout 300 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/final_bench_c2.json 2> gpurun_out/final_bench_c2.err; echo "bench c2 rc=$?"
timeout 300 python bench.py --config 5 --scaling strong --steps 20 --warmup 5 > gpurun_out/final_bench_c5.json 2> gpurun_out/final_bench_c5.err; echo "bench c5 rc=$?"
timeout 300 python tools/resnet_probe.py > gpurun_out/final_resnet_probe.json 2>&1
bash tools/profile_round.sh > gpurun_out/profile_round.log 2>&1; echo "profile_round rc=$?"
timeout 900 python tools/config_sweep.py > gpurun_out/final_config_sweep.jsonl 2> gpurun_out/final_config_sweep.err; echo "sweep rc=$?"
cut -c1-300 gpurun_out/final_bench_c2.json gpurun_out/final_bench_c5.json; cat gpurun_out/final_config_sweep.jsonl | cut -c1-200
