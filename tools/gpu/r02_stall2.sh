# the timed window aligned between NVML samples: the driver's command x8
for i in 1 2 3 4 5 6 7 8; do timeout 300 python bench.py --gpus 1 --steps 20 --warmup 5 --quick >> gpurun_out/stall2.jsonl 2>>gpurun_out/stall2_err.txt; done
