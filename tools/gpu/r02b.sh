for i in 1 2; do timeout 200 python tools/trace_window.py steps=20 > gpurun_out/r02b_tw20_$i.txt 2>&1; done
timeout 200 python tools/trace_window.py steps=100 > gpurun_out/r02b_tw100.txt 2>&1
tail -3 gpurun_out/r02b_tw20_1.txt
