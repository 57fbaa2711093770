# Kernel role cycle counters (PROTEA_DBG build) over 7 heavy lock-step iterations of config 2 (tools/dbg_counters.py heavy)
PROTEA_DBG=1 python paper_2207_01053_b200/build.py > /dev/null && timeout 200 python tools/dbg_counters.py heavy > gpurun_out/dbg_heavy.txt 2>&1
cat gpurun_out/dbg_heavy.txt
