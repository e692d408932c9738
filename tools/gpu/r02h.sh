timeout 200 python tools/lone_trace.py > gpurun_out/r02h_lone400.txt 2>&1
timeout 200 python tools/lone_trace.py split_pct=120 > gpurun_out/r02h_lone120.txt 2>&1
