# the timed window started late between two NVML samples (offset 0.75 / 0.5 of the period)
for i in 1 2 3 4 5 6; do
  echo 0.75 >> gpurun_out/stall3_tags.txt; timeout 300 python bench.py --gpus 1 --steps 20 --warmup 5 --quick >> gpurun_out/stall3.jsonl 2>>gpurun_out/stall3_err.txt
  echo 0.5 >> gpurun_out/stall3_tags.txt; GMX_CLOCK_OFFSET=0.5 timeout 300 python bench.py --gpus 1 --steps 20 --warmup 5 --quick >> gpurun_out/stall3.jsonl 2>>gpurun_out/stall3_err.txt
done
