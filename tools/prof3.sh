PROTEA_DBG=1 python paper_2207_01053_b200/build.py > /dev/null && timeout 200 python tools/dbg_counters.py heavy > gpurun_out/dbg_heavy.txt 2>&1
cat gpurun_out/dbg_heavy.txt
