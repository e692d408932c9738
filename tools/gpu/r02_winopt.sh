# 20-round resident window (tools/window_fixed.py, medians of 15) under skew-window / grab options
for o in "" "resident_window=32" "resident_window=64" "grab_ahead=2" "resident_window=8"; do echo "=== $o"; timeout 300 python tools/window_fixed.py $o; done > gpurun_out/winopt.txt 2>&1
