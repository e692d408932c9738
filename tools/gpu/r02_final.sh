# final validation of the round: GPU tests, smoke, the driver's command x3, reference arm
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/final_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/final_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/final_smoke.log
for i in 1 2 3; do timeout 300 python bench.py --gpus 1 --steps 20 --warmup 5 >> gpurun_out/final_bench.jsonl 2>>gpurun_out/final_bench_err.txt; done
timeout 300 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 >> gpurun_out/final_bench_ref.jsonl 2>>gpurun_out/final_bench_err.txt
