timeout 200 python tools/chain_latency.py bert_base resident=1 > gpurun_out/r02s.txt 2>&1
timeout 200 python tools/chain_latency.py bert_base resident=0 >> gpurun_out/r02s.txt 2>&1
