for cfg in "prestep=1 delay_us=200" "prestep=0 delay_us=200" "prestep=1 delay_us=200 split_pct=120"; do
echo "== $cfg" >> gpurun_out/r02f.txt
timeout 200 python tools/trace_window.py steps=20 $cfg > /tmp/tw.txt 2>&1
grep -E "^window|^    0 |^    1 |^    2 |^    3 |^   19 |^held" /tmp/tw.txt >> gpurun_out/r02f.txt
grep -A4 -E "^step [0-3]:" /tmp/tw.txt | grep -E "epi done|^step" >> gpurun_out/r02f.txt
done
