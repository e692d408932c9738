timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/r02u_test.txt
timeout 200 python tools/lone_trace.py 2>&1 | head -3 > gpurun_out/r02u.txt
for i in 1 2; do timeout 200 python tools/trace_window.py steps=20 > /tmp/tw.txt 2>&1; grep -E "^window|^    0 |^   19 |^held" /tmp/tw.txt >> gpurun_out/r02u.txt; done
timeout 200 python tools/chain_latency.py bert_base resident=1 >> gpurun_out/r02u.txt 2>&1
