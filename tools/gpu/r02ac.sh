timeout 300 python -m pytest tests/test_exec_gpu.py -m gpu -x -q -k tun 2>&1 | tail -2 > gpurun_out/r02ac.txt
for st in 0 1; do for rows in 16 64 2368 4000; do
timeout 100 python tools/gemv_ingest.py $rows gemv_staged=$st 2>&1 | tail -2 | sed "s/^/staged=$st /" >> gpurun_out/r02ac.txt
done; done
