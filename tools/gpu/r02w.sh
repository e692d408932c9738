timeout 300 python tools/instr_resident.py > gpurun_out/r02w.txt 2>&1
