python -m pytest tests -m gpu -q -x -k "not all_views" > gpurun_out/r2c_pytest_gpu.txt 2>&1; echo "rc=$?" >> gpurun_out/r2c_pytest_gpu.txt
tail -30 gpurun_out/r2c_pytest_gpu.txt
