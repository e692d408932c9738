for sp in 400 200 120 80; do for i in 1 2; do
echo "== split_pct=$sp run $i" >> gpurun_out/r02d.txt
timeout 200 python tools/trace_window.py steps=20 split_pct=$sp > /tmp/tw.txt 2>&1
grep -E "^window|^held|^    0 |^   19 " /tmp/tw.txt >> gpurun_out/r02d.txt
grep -A4 "^step 0" /tmp/tw.txt | grep "epi done" >> gpurun_out/r02d.txt
done; done
