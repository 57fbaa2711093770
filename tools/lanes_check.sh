# lanes experiment: correctness (bf16 tests with PROTEA_LANES=2) and config-2 / config-3 round time
PROTEA_LANES=2 timeout 300 python -m pytest tests -m gpu -x -q --timeout 120 -k "bf16 or determinism or virtual" 2>&1 | tail -2
for L in 1 2 3; do
  PROTEA_LANES=$L timeout 200 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_l$L.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/bench_l$L.json'));print('lanes', $L, d['ms_per_step'], d['value'])"
  PROTEA_LANES=$L timeout 100 python tools/config_probe.py 3 | cut -c1-80
done
