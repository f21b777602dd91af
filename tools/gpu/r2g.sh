ncu --set full --clock-control none --import-source on -k regex:k_resample_window -s 2 -c 1 -o gpurun_out/r2g_win python bench.py --only --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/r2g_ncu.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/r2g_ncu.log
