python -m pytest tests -m gpu -q -x -k "not all_views" > gpurun_out/r2f_pytest_gpu.txt 2>&1; echo "rc=$?" >> gpurun_out/r2f_pytest_gpu.txt
tail -4 gpurun_out/r2f_pytest_gpu.txt
for W in 1 0; do
CBN_WINDOW_GATHER=$W timeout 600 python bench.py --only --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2f_bench_w$W.json 2> gpurun_out/r2f_bench_w$W.err
echo "bench W=$W rc=$?"; tail -3 gpurun_out/r2f_bench_w$W.err
done
