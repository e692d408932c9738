# round-2 evidence (final kernel): launch list + one full capture of the C2 coalesced kernel, then bench lines
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r02b.csv python bench.py --launch-per-step --steps 20 --warmup 3 --quick > gpurun_out/ncu_l_r02b.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:coalesced -s 20 -c 1 -f -o gpurun_out/prof_r02b python tools/ncu_target.py c2 20 1 > gpurun_out/ncu_f_r02b.log 2>&1
for i in 1 2 3; do timeout 300 python bench.py --gpus 1 --steps 20 --warmup 5 >> gpurun_out/bench_r02c.jsonl 2>>gpurun_out/bench_r02c_err.txt; done
timeout 300 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_r02c_ref.jsonl 2>&1
