cd $GRAFT_REPO_ROOT
timeout 600 python tools/bigbatch_diag.py > gpurun_out/bigbatch_diag.jsonl 2> gpurun_out/bigbatch_diag.err
tail -2 gpurun_out/bigbatch_diag.err
timeout 1500 python -m pytest tests/test_gpu_bigbatch.py tests/test_gpu_evaluate_round.py tests/test_gpu_teacher_forced.py tests/test_gpu_tc.py tests/test_gpu_parity.py -q --timeout 900 2>&1 | tail -40 > gpurun_out/t_new.log
tail -8 gpurun_out/t_new.log
timeout 300 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_t.json 2> gpurun_out/bench_t.err
python -c "
import json; d=json.load(open('gpurun_out/bench_t.json')); print(d['value'], d['ms_per_step'], d['roofline']['kernel'], d['roofline']['frac'], d['roofline'].get('implementation_extra'))"
tail -3 gpurun_out/bench_t.err
