timeout 300 python -m pytest tests/test_exec_gpu.py -m gpu -x -q 2>&1 | tail -2 > gpurun_out/r02af.txt
for i in 1 2; do for so in _ab/prev/libgmx_exec.so _ab/inl/libgmx_exec.so paper_1901_10008_b200/lib/libgmx_exec.so; do
timeout 200 python tools/ab_held.py $so >> gpurun_out/r02af.txt 2>&1
done; done
timeout 200 python tools/c1_kernel.py gemv_staged=1 2>&1 | head -1 >> gpurun_out/r02af.txt
timeout 200 python tools/c1_kernel.py _ab/inl/libgmx_exec.so gemv_staged=1 2>&1 | head -1 >> gpurun_out/r02af.txt
