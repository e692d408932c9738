# lone-step breakdown of the C2 coalesced step under a few per-step split settings
for o in "" "split_pct_step=100" "split_pct_step=400"; do echo "=== $o"; timeout 300 python tools/lone_trace.py $o; done > gpurun_out/lone_r02i.txt 2>&1
