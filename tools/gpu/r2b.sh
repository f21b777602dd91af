set -x
python -m pytest tests/test_gpu_bins.py tests/test_gpu_cli_default.py tests/test_gpu_config2.py -q -k "not all_views" > gpurun_out/r2b_pytest_new.txt 2>&1; echo "rc=$?" >> gpurun_out/r2b_pytest_new.txt
tail -40 gpurun_out/r2b_pytest_new.txt
