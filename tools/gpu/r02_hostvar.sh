# run-to-run variance of the serving loop on one box: 5 quick bench runs
for i in 1 2 3 4 5; do timeout 300 python bench.py --gpus 1 --steps 20 --warmup 5 --quick >> gpurun_out/hostvar.jsonl 2>>gpurun_out/hostvar_err.txt; done
nproc >> gpurun_out/hostvar_err.txt; cat /proc/cpuinfo | grep "model name" | head -1 >> gpurun_out/hostvar_err.txt; uptime >> gpurun_out/hostvar_err.txt
