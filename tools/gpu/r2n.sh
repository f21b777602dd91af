python -m pytest tests -m gpu -q -x > gpurun_out/r2n_pytest_gpu.txt 2>&1; echo "rc=$?" >> gpurun_out/r2n_pytest_gpu.txt; tail -3 gpurun_out/r2n_pytest_gpu.txt
python tools/parity_report.py > gpurun_out/r2n_parity.txt 2>&1; echo "parity rc=$?"; tail -40 gpurun_out/r2n_parity.txt
