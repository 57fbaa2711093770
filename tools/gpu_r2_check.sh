cd $GRAFT_REPO_ROOT
timeout 300 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_t.json 2> gpurun_out/bench_t.err
python -c "
import json; d=json.load(open('gpurun_out/bench_t.json')); print(d['value'], d['ms_per_step'], d['roofline']['kernel'], d['roofline']['frac'], d['roofline']['per_launch']['avg_ns'], d['detail']['op_ms_warmup'])"
tail -3 gpurun_out/bench_t.err
timeout 900 python -m pytest tests/test_gpu_tc.py -q --timeout 600 -k "one_step or deterministic or config2_bf16" 2>&1 | tail -3
