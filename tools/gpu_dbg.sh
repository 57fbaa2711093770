cd $GRAFT_REPO_ROOT
for i in 1 2; do
  timeout 600 python -m pytest tests -m gpu -q --timeout 300 -k "resnet or config5 or r8" 2>&1 | grep -E "passed|failed|FAILED|Error:" | head -5 | sed "s/^/run$i: /"
done
timeout 300 python tools/resnet_probe.py 2>&1 | cut -c1-400
