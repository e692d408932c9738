timeout 120 python tools/sm_ingest.py > gpurun_out/r02i.txt 2>&1
timeout 120 python tools/sm_ingest.py 512 128 4608 >> gpurun_out/r02i.txt 2>&1
timeout 120 python tools/sm_ingest.py 128 49 8192 >> gpurun_out/r02i.txt 2>&1
