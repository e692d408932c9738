# the driver's 20-step window under resident plan options, 3 runs each on one box
for o in "" "--exec-opt split_pct=200" "--exec-opt split_pct=100" "--exec-opt grab_ahead=0" "--exec-opt resident_window=4" "--exec-opt split_pct=800"; do
  for i in 1 2 3; do echo "$o" >> gpurun_out/winsweep_tags.txt; timeout 300 python bench.py --gpus 1 --steps 20 --warmup 5 --quick $o >> gpurun_out/winsweep.jsonl 2>>gpurun_out/winsweep_err.txt; done
done
