# round-2 evidence for the final build: launch list + one full capture of the C2 coalesced kernel
# (summarised here with tools/ncu_summary.py gpurun_out/prof_r02i.ncu-rep gpurun_out/launches_r02i.csv profiles/r02i_c2)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r02i.csv python bench.py --launch-per-step --steps 20 --warmup 3 --quick > gpurun_out/ncu_l_r02i.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:coalesced -s 20 -c 1 -f -o gpurun_out/prof_r02i python tools/ncu_target.py c2 20 1 > gpurun_out/ncu_f_r02i.log 2>&1
