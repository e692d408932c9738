for rows in 16 2368 4000; do
timeout 100 python tools/gemv_ingest.py $rows 2>&1 | tail -1 >> gpurun_out/r02ad.txt
done
timeout 200 python tools/c1_kernel.py _ab/prev/libgmx_exec.so 2>&1 | head -1 >> gpurun_out/r02ad.txt
timeout 200 python tools/c1_kernel.py 2>&1 | head -1 >> gpurun_out/r02ad.txt
timeout 200 python tools/ab_held.py _ab/prev/libgmx_exec.so >> gpurun_out/r02ad.txt 2>&1
timeout 200 python tools/ab_held.py >> gpurun_out/r02ad.txt 2>&1
