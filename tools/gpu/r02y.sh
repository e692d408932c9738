timeout 300 python -m pytest tests/test_exec_gpu.py -m gpu -x -q 2>&1 | tail -2 > gpurun_out/r02y.txt
for i in 1 2 3; do
timeout 200 python tools/ab_held.py _ab/prev/libgmx_exec.so >> gpurun_out/r02y.txt 2>&1
timeout 200 python tools/ab_held.py >> gpurun_out/r02y.txt 2>&1
done
