# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_run.py (GPU box); logs -> gpurun_out/
cd $GRAFT_REPO_ROOT
for tool in memcheck synccheck racecheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_run.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_rc.txt
  tail -3 gpurun_out/sanitize_$tool.log
done
