# config-5 round time vs the ResNet-8 dgrad || wgrad overlap threshold (rows), final code
cd $GRAFT_REPO_ROOT
for R in 256 512 1024 2048 4096 100000; do
  PROTEA_R8_OVERLAP_ROWS=$R timeout 300 python tools/host_probe.py 5 2>&1 | tail -n 1 | sed "s/^/r8_overlap_rows=$R: /"
done
PROTEA_R8_OVERLAP=0 timeout 300 python tools/host_probe.py 5 2>&1 | tail -n 1 | sed "s/^/r8_overlap=0: /"
