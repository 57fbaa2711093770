timeout 600 python -m pytest tests -m gpu -x -q --timeout 120 2>&1 | tail -5 > gpurun_out/gpu_t.log
timeout 240 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_t.json 2> gpurun_out/bench_t.err
cat gpurun_out/gpu_t.log
python - <<'PY'
import json
d=json.load(open("gpurun_out/bench_t.json"))
print(d["value"], d["ms_per_step"], d["roofline"]["kernel"], d["roofline"]["frac"])
print({k: round(v, 2) for k, v in d["detail"]["op_ms_warmup"].items()})
PY
timeout 300 python tools/tail_probe.py > gpurun_out/tail.json 2> gpurun_out/tail.err; cat gpurun_out/tail.json
