# fc1-wgrad deferral threshold sweep (rows per lock-step iteration)
for R in 0 640 2000 100000; do
  PROTEA_OVERLAP_ROWS=$R timeout 240 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_ov$R.json 2> gpurun_out/bench_ov$R.err
  python -c "import json;d=json.load(open('gpurun_out/bench_ov$R.json'));print($R, d['ms_per_step'], d['value'])"
done
