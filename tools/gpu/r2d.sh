python -m pytest tests -m gpu -q -x -k "not all_views" > gpurun_out/r2d_pytest_gpu.txt 2>&1; echo "rc=$?" >> gpurun_out/r2d_pytest_gpu.txt
tail -5 gpurun_out/r2d_pytest_gpu.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2d_bench.json 2> gpurun_out/r2d_bench.err
echo "bench rc=$?"; tail -5 gpurun_out/r2d_bench.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2d_ref.json 2> gpurun_out/r2d_ref.err
echo "ref rc=$?"; tail -3 gpurun_out/r2d_ref.err
