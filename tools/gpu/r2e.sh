timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2e_bench.json 2> gpurun_out/r2e_bench.err
echo "bench rc=$?"; tail -5 gpurun_out/r2e_bench.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2e_ref.json 2> gpurun_out/r2e_ref.err
echo "ref rc=$?"; tail -3 gpurun_out/r2e_ref.err
