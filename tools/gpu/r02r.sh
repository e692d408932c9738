timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/r02r_test.txt
timeout 200 python tools/chain_latency.py resnet50 resident=1 > gpurun_out/r02r.txt 2>&1
timeout 200 python tools/chain_latency.py bert_base resident=1 >> gpurun_out/r02r.txt 2>&1
timeout 200 python tools/trace_window.py steps=20 > /tmp/tw.txt 2>&1; grep -E "^window|^    0 |^   19 |^held" /tmp/tw.txt >> gpurun_out/r02r.txt
for i in 1 2; do timeout 300 python bench.py --gpus 1 --steps 20 --warmup 5 >> gpurun_out/r02r_bench.jsonl 2>gpurun_out/r02r_bench_err.txt; done
