timeout 200 python tools/lone_trace.py > gpurun_out/r02o_lone400.txt 2>&1
timeout 200 python tools/lone_trace.py split_pct=120 > gpurun_out/r02o_lone120.txt 2>&1
timeout 200 python tools/lone_trace.py split_pct=60 > gpurun_out/r02o_lone60.txt 2>&1
