
python tools/probe/e2e_timeline.py > gpurun_out/r2l_tl.txt 2>&1; tail -5 gpurun_out/r2l_tl.txt

