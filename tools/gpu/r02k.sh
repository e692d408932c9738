timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/r02k_test.txt
timeout 120 python tools/sm_ingest.py | head -2 > gpurun_out/r02k.txt 2>&1
timeout 120 python tools/sm_ingest.py 128 256 4608 | head -2 >> gpurun_out/r02k.txt 2>&1
timeout 200 python tools/lone_trace.py 2>&1 | head -3 >> gpurun_out/r02k.txt
timeout 200 python tools/lone_trace.py split_pct=120 2>&1 | head -3 >> gpurun_out/r02k.txt
timeout 200 python tools/trace_window.py steps=20 > /tmp/tw.txt 2>&1; grep -E "^window|^    0 |^   19 |^held" /tmp/tw.txt >> gpurun_out/r02k.txt
for i in 1 2; do timeout 300 python bench.py --gpus 1 --steps 20 --warmup 5 >> gpurun_out/r02k_bench.jsonl 2>gpurun_out/r02k_bench_err.txt; done
