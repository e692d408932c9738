timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/r02n_test.txt
for ga in 0 1 2 64; do
echo "== grab_ahead=$ga" >> gpurun_out/r02n.txt
timeout 200 python tools/trace_window.py steps=20 grab_ahead=$ga > /tmp/tw.txt 2>&1
grep -E "^window|^held|^    0 |^   19 |Error|error" /tmp/tw.txt >> gpurun_out/r02n.txt
grep -A6 "^step 0:" /tmp/tw.txt | grep -E "items done|prod issued" >> gpurun_out/r02n.txt
done
