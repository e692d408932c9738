timeout 300 python -m pytest tests/test_exec_gpu.py -m gpu -x -q 2>&1 | tail -2 > gpurun_out/r02ae.txt
for st in 0 1; do for rows in 16 2368; do
timeout 100 python tools/gemv_ingest.py $rows gemv_staged=$st 2>&1 | tail -1 | sed "s/^/staged=$st /" >> gpurun_out/r02ae.txt
done; done
timeout 200 python tools/c1_kernel.py 2>&1 | head -1 >> gpurun_out/r02ae.txt
timeout 200 python tools/c1_kernel.py gemv_staged=1 2>&1 | head -1 >> gpurun_out/r02ae.txt
timeout 200 python tools/ab_held.py _ab/prev/libgmx_exec.so >> gpurun_out/r02ae.txt 2>&1
timeout 200 python tools/ab_held.py >> gpurun_out/r02ae.txt 2>&1
