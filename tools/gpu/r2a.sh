set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -x -q > gpurun_out/r2a_pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/r2a_pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2a_smoke.txt 2>&1
python bench.py --steps 20 --warmup 5 > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err
python bench.py --steps 20 --warmup 5 --direction back --no-cpu-baseline > gpurun_out/r2a_bench_back.json 2>> gpurun_out/r2a_bench.err
tail -3 gpurun_out/r2a_pytest_gpu.txt; cat gpurun_out/r2a_smoke.txt
