python -m pytest tests/test_gpu_config2.py -q -k "all_views" > gpurun_out/r2m_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/r2m_pytest.txt; tail -5 gpurun_out/r2m_pytest.txt
