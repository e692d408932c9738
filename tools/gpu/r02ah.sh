timeout 300 python -m pytest tests/test_exec_gpu.py -m gpu -x -q -k long_lists 2>&1 | tail -30 > gpurun_out/r02ah.txt
timeout 300 python -m pytest tests/test_exec_gpu.py -m gpu -x -q -k long_lists 2>&1 | tail -3 >> gpurun_out/r02ah.txt
