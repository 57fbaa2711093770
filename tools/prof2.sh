timeout 300 python tools/tail_probe.py > gpurun_out/tail.json 2> gpurun_out/tail.err; cat gpurun_out/tail.json; tail -3 gpurun_out/tail.err
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/round_launches.csv python tools/prof_round.py > gpurun_out/round_launches.log 2>&1
ls -la gpurun_out
