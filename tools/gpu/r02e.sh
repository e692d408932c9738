for d in 0 100 1000; do
echo "== delay_us=$d" >> gpurun_out/r02e.txt
timeout 200 python tools/trace_window.py steps=20 delay_us=$d > /tmp/tw.txt 2>&1
grep -E "^window|^    0 |^    1 |^    2 |^   19 " /tmp/tw.txt >> gpurun_out/r02e.txt
grep -A4 "^step 0" /tmp/tw.txt | grep "epi done" >> gpurun_out/r02e.txt
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:coalesced -s 20 -c 1 -f -o gpurun_out/prof_r02e python tools/ncu_target.py c2 20 1 > gpurun_out/ncu_r02e.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:coalesced -s 0 -c 1 -f -o gpurun_out/prof_r02e_first python tools/ncu_target.py c2 0 1 > gpurun_out/ncu_r02e_first.log 2>&1
