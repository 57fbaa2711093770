cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests -m gpu -q --timeout 1200 2>&1 | tail -30 > gpurun_out/t_all.log
grep -E "passed|failed|^FAILED" gpurun_out/t_all.log | tail -10
timeout 300 python bench.py --config 5 --scaling strong --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
python -c "
import json; d=json.load(open('gpurun_out/bench_c5.json')); print('c5', d['value'], d['ms_per_step'], d['roofline']['kernel'], d['roofline']['frac'], d['config']['workload'])"
tail -2 gpurun_out/bench_c5.err
timeout 1500 python tools/paper_arms_r2.py > gpurun_out/paper_arms_r2.json 2> gpurun_out/paper_arms_r2.err
tail -5 gpurun_out/paper_arms_r2.err
