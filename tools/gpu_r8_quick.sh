# ResNet-8 check: parity / HWM tests touching config 5 / ResNet-8, then the per-op probe
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 300 -k "resnet or config5 or r8 or hwm" > gpurun_out/r8_tests.log 2>&1; echo "tests rc=$?"
tail -n 3 gpurun_out/r8_tests.log
timeout 300 python tools/resnet_probe.py > gpurun_out/resnet_probe.json 2>&1; echo "probe rc=$?"
cat gpurun_out/resnet_probe.json | cut -c1-700
timeout 300 python tools/host_probe.py 5 2>&1 | tail -n 2
timeout 300 python bench.py --config 5 --scaling strong --steps 20 --warmup 5 > gpurun_out/final_bench_c5.json 2> gpurun_out/final_bench_c5.err; echo "bench c5 rc=$?"
cut -c1-300 gpurun_out/final_bench_c5.json; tail -n 2 gpurun_out/final_bench_c5.err
