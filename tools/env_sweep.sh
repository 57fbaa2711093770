# Round time (config 2 and config 5, bf16, 1 GPU) under launch-configuration knobs
cd $GRAFT_REPO_ROOT
for E in "X=0" "PROTEA_PDL=1" "PROTEA_LANES=2" "PROTEA_PDL=1 PROTEA_LANES=2" "PROTEA_R8_OVERLAP=0"; do
  for c in 5 2; do
    env $E timeout 300 python tools/host_probe.py $c 2>&1 | tail -n 1 | sed "s/^/$E: /"
  done
done
