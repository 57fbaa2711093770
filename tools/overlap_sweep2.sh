# config-2 round time vs the light-iteration fc1 wgrad deferral threshold (rows), final code
cd $GRAFT_REPO_ROOT
for R in 0 300 640 1000 1500; do
  PROTEA_OVERLAP_ROWS=$R timeout 300 python tools/host_probe.py 2 2>&1 | tail -n 1 | sed "s/^/overlap_rows=$R: /"
done
