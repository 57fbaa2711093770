# ResNet-8 dgrad/wgrad overlap threshold (rows per lock-step iteration): config 5 at 1 and 8-GPU shares
for R in 0 1024 2048 4096 100000; do
  echo "== rows <= $R"
  PROTEA_R8_OVERLAP_ROWS=$R timeout 200 python tools/config_sweep.py 5 | python -c "
import json,sys
for l in sys.stdin: r=json.loads(l); print(r['gpus'], round(r['round_ms'],2))"
done
