set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/r02a_gputest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02a_smoke.txt 2>&1
for i in 1 2 3; do timeout 300 python bench.py --gpus 1 --steps 20 --warmup 5 >> gpurun_out/r02a_bench.jsonl 2>gpurun_out/r02a_bench_err.txt; done
timeout 300 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02a_ref.jsonl 2>&1
cat gpurun_out/r02a_gputest.txt
