for i in 1 2; do
timeout 200 python tools/ab_held.py >> gpurun_out/r02x.txt 2>&1
timeout 200 python tools/ab_held.py dbg=8 >> gpurun_out/r02x.txt 2>&1
done
