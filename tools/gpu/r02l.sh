for sp in 400 200 120; do for i in 1 2; do
echo "== split_pct=$sp run $i" >> gpurun_out/r02l.txt
timeout 200 python tools/trace_window.py steps=20 split_pct=$sp > /tmp/tw.txt 2>&1
grep -E "^window|^held|^    0 |^   19 " /tmp/tw.txt >> gpurun_out/r02l.txt
done; done
