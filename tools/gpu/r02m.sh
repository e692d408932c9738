timeout 200 python tools/trace_window.py steps=20 > gpurun_out/r02m_a.txt 2>&1
timeout 200 python tools/trace_window.py steps=20 prestep=1 delay_us=200 > gpurun_out/r02m_b.txt 2>&1
