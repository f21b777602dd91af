python tools/probe/sanitize_case.py > gpurun_out/r2o_plain.txt 2>&1 && \
timeout 1500 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 9 python tools/probe/sanitize_case.py > gpurun_out/r2o_memcheck.txt 2>&1
echo "memcheck rc=$?"; tail -8 gpurun_out/r2o_memcheck.txt
