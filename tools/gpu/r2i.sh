python -m pytest tests/test_gpu_config2.py tests/test_gpu_projector.py -q -x -k "not all_views" > gpurun_out/r2i_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/r2i_pytest.txt; tail -2 gpurun_out/r2i_pytest.txt
timeout 600 python bench.py --only --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2i_bench.json 2> gpurun_out/r2i_bench.err && \
ncu --set full --clock-control none --import-source on -k regex:k_resample_window -s 2 -c 1 -o gpurun_out/r2i_win python bench.py --only --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/r2i_ncu.log 2>&1
echo "rc=$?"
