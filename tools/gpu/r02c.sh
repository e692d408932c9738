timeout 200 python tools/trace_window.py steps=20 > gpurun_out/r02c_tw20.txt 2>&1
