# HEAD state: full GPU suite, config-2 bench, config-5 strong bench, ResNet-8 probe.
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -n 5 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "bench2 rc=$?"
timeout 300 python bench.py --config 5 --scaling strong --steps 5 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "bench5 rc=$?"
timeout 300 python tools/resnet_probe.py > gpurun_out/resnet_probe.json 2>&1; echo "probe rc=$?"
cut -c1-600 gpurun_out/bench_c2.json gpurun_out/bench_c5.json gpurun_out/resnet_probe.json
