# deferred fc1 wgrad occupancy sweep (dynamic smem floor -> CTAs per SM)
for S in 0 60000 100000 200000; do
  PROTEA_F1W_SIDE_SMEM=$S timeout 200 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_fs$S.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/bench_fs$S.json'));print($S, d['ms_per_step'], d['value'])"
done
