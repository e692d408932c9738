for i in 1 2 3; do
timeout 200 python tools/ab_held.py _ab/prev/libgmx_exec.so >> gpurun_out/r02v.txt 2>&1
timeout 200 python tools/ab_held.py >> gpurun_out/r02v.txt 2>&1
done
