# config-2 quick check: full GPU suite, bench line, tail probe (live per-iteration op cost)
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -n 2 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "bench2 rc=$?"
cut -c1-300 gpurun_out/bench_c2.json
timeout 300 python tools/tail_probe.py > gpurun_out/tail.json 2>&1
cat gpurun_out/tail.json | cut -c1-600
