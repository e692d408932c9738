# latency plans for resident steps entering an idle device (split_pct_idle): GPU tests, window sweep, window trace
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/idle_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/idle_pytest.log
for i in 1 2 3; do
  for o in "" "--exec-opt split_pct_idle=0" "--exec-opt split_pct_idle=200" "--exec-opt split_pct_idle=50"; do
    echo "$o" >> gpurun_out/idle_tags.txt; timeout 300 python bench.py --gpus 1 --steps 20 --warmup 5 --quick $o >> gpurun_out/idle.jsonl 2>>gpurun_out/idle_err.txt
  done
done
timeout 300 python tools/trace_window.py > gpurun_out/idle_trace.txt 2>&1
