for i in 1 2; do for sp in 400 300 250 200; do
echo "== split_pct=$sp" >> gpurun_out/r02ab.txt
timeout 200 python tools/trace_window.py steps=20 split_pct=$sp > /tmp/tw.txt 2>&1
grep -E "^window|^held" /tmp/tw.txt >> gpurun_out/r02ab.txt
done; done
