set -x
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r01f.csv python bench.py --launch-per-step --steps 20 --warmup 3 --quick > gpurun_out/ncu_l.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:coalesced -s 12 -c 1 -f -o gpurun_out/prof_r01f python bench.py --launch-per-step --steps 5 --warmup 3 --quick > gpurun_out/ncu_f.log 2>&1
ls -la gpurun_out/
