timeout 300 python tools/c4_poisson.py --tenants 3 --rates 5 --duration-ms 300 --stagger-ns 3000 > gpurun_out/r02p_c4small.jsonl 2>&1
timeout 300 python tools/c4_poisson.py --tenants 3 --rates 5 --duration-ms 300 --stagger-ns 3000 --resident >> gpurun_out/r02p_c4small.jsonl 2>&1
timeout 600 python tools/c4_poisson.py --rates 2,5,10 --stagger-ns 3000 > gpurun_out/r02p_c4.jsonl 2>&1
timeout 600 python tools/c4_poisson.py --rates 2,5,10 --stagger-ns 3000 --resident >> gpurun_out/r02p_c4.jsonl 2>&1
