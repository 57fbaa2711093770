cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -k "hwm or tc or teacher" > gpurun_out/last_tests.log 2>&1; echo "tests rc=$?"
tail -n 2 gpurun_out/last_tests.log; grep -E "^FAILED|Error" gpurun_out/last_tests.log | head -5
timeout 300 python tools/tail_probe.py 2>&1 | cut -c1-420
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "bench2 rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/bench_c2.json').read().strip().splitlines()[-1]); r=d['roofline']; print(d['value'], d['ms_per_step'], r['achieved'], r['frac'])"
