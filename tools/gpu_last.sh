cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/last_tests.log 2>&1; echo "tests rc=$?"
tail -n 2 gpurun_out/last_tests.log; grep -E "^FAILED|Error" gpurun_out/last_tests.log | head -5
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo "smoke rc=$?"
timeout 300 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/final_bench_c2.json 2> gpurun_out/final_bench_c2.err; echo "bench c2 rc=$?"
timeout 300 python tools/tail_probe.py > gpurun_out/final_tail.json 2>&1
python -c "
import json
for f in ['gpurun_out/final_bench_c2.json']:
    d=json.loads(open(f).read().strip().splitlines()[-1]); r=d['roofline']
    print(f, d['value'], d['ms_per_step'], d['e2e']['value'], r['kernel'], r['frac'], r['per_launch']['launches'], d['clocks'])
"
cut -c1-300 gpurun_out/final_tail.json
