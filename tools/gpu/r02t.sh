timeout 200 python tools/c1_kernel.py > gpurun_out/r02t.txt 2>&1
timeout 200 python tools/c1_kernel.py gemv_staged=1 >> gpurun_out/r02t.txt 2>&1
timeout 300 python tools/configs.py --configs c1 >> gpurun_out/r02t.txt 2>&1
