# host state before the timed window: committed settle (A), busy-aligned between NVML samples (B), 20 ms host spin (C)
for i in 1 2 3 4 5 6; do
  echo A >> gpurun_out/stall4_tags.txt; timeout 300 python bench.py --gpus 1 --steps 20 --warmup 5 --quick >> gpurun_out/stall4.jsonl 2>>gpurun_out/stall4_err.txt
  echo B >> gpurun_out/stall4_tags.txt; GMX_CLOCK_ALIGN=1 timeout 300 python bench.py --gpus 1 --steps 20 --warmup 5 --quick >> gpurun_out/stall4.jsonl 2>>gpurun_out/stall4_err.txt
  echo C >> gpurun_out/stall4_tags.txt; timeout 300 python bench.py --gpus 1 --steps 20 --warmup 5 --quick --host-spin-ms 20 >> gpurun_out/stall4.jsonl 2>>gpurun_out/stall4_err.txt
done
