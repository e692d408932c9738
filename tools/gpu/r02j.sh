echo "== base" > gpurun_out/r02j.txt; timeout 120 python tools/sm_ingest.py | head -4 >> gpurun_out/r02j.txt 2>&1
echo "== dbg=4 (no MMA)" >> gpurun_out/r02j.txt; timeout 120 python tools/sm_ingest.py dbg=4 | head -4 >> gpurun_out/r02j.txt 2>&1
echo "== promo 0" >> gpurun_out/r02j.txt; GMX_L2_PROMO=0 timeout 120 python tools/sm_ingest.py | head -4 >> gpurun_out/r02j.txt 2>&1
echo "== promo 128" >> gpurun_out/r02j.txt; GMX_L2_PROMO=128 timeout 120 python tools/sm_ingest.py | head -4 >> gpurun_out/r02j.txt 2>&1
echo "== 128x256x4608" >> gpurun_out/r02j.txt; timeout 120 python tools/sm_ingest.py 128 256 4608 | head -4 >> gpurun_out/r02j.txt 2>&1
