CBN_LIB=check python tools/probe/sanitize_case.py > gpurun_out/r2bq_check_case.txt 2>&1; echo "case rc=$?" >> gpurun_out/r2bq_check_case.txt; tail -3 gpurun_out/r2bq_check_case.txt
CBN_LIB=check timeout 1500 python -m pytest tests -m gpu -q -x -k "not all_views" --ignore=tests/test_gpu_comm.py > gpurun_out/r2bq_check_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/r2bq_check_pytest.txt; tail -3 gpurun_out/r2bq_check_pytest.txt
CBN_LIB=check timeout 900 python bench.py --only --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2bq_check_bench_fwd.json 2>&1; echo "fwd rc=$?"
CBN_LIB=check timeout 900 python bench.py --only --direction back --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2bq_check_bench_bp.json 2>&1; echo "bp rc=$?"
CBN_LIB=check CBN_C4_POINTS=20000000 timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2bq_check_bench_c4.json 2>&1; echo "c4 rc=$?"
