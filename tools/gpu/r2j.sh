python tools/probe/e2e_breakdown.py > gpurun_out/r2j_e2e.txt 2>&1; tail -5 gpurun_out/r2j_e2e.txt; nproc; cat /sys/kernel/mm/transparent_hugepage/enabled
