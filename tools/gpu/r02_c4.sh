# C4 with the final build: latency plans on (default) and off, stagger 1 us
for i in 1 2; do
timeout 600 python tools/c4_poisson.py --resident --rates 2,5,10 --stagger-ns 1000 >> gpurun_out/c4_r02i.jsonl 2>>gpurun_out/c4_err.txt
timeout 600 python tools/c4_poisson.py --resident --rates 2,5,10 --stagger-ns 1000 --opt split_pct_idle=0 >> gpurun_out/c4_r02i_idle0.jsonl 2>>gpurun_out/c4_err.txt
done
