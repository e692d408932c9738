# host stalls in the timed window: with / without the NVML sampler, interrupts per core
grep -i -E "nvidia|CPU0" /proc/interrupts | cut -c1-250 > gpurun_out/stall_irq.txt
for i in 1 2 3 4 5 6; do
  echo default >> gpurun_out/stall_tags.txt; timeout 300 python bench.py --gpus 1 --steps 20 --warmup 5 --quick >> gpurun_out/stall.jsonl 2>>gpurun_out/stall_err.txt
  echo noclocks >> gpurun_out/stall_tags.txt; GMX_BENCH_CLOCKS=0 timeout 300 python bench.py --gpus 1 --steps 20 --warmup 5 --quick >> gpurun_out/stall.jsonl 2>>gpurun_out/stall_err.txt
done
grep -i -E "nvidia|CPU0" /proc/interrupts | cut -c1-250 >> gpurun_out/stall_irq.txt
