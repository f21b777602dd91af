#!/bin/bash
# One GPU session: tests, smoke, bench, launch list, ncu captures -> gpurun_out/$TAG
TAG=${1:-r1}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -m pytest tests -q -m gpu 2>&1 | tail -3 > $OUT/pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1; echo "smoke rc=$?" >> $OUT/smoke.txt
python bench.py > $OUT/bench.json 2> $OUT/bench.err
python bench.py --direction back --no-cpu-baseline > $OUT/bench_back.json 2> $OUT/bench_back.err
python bench.py --config 4 --steps 5 > $OUT/bench_c4.json 2> $OUT/bench_c4.err
python tools/profile_step.py > $OUT/plain.log 2>&1 && \
ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $OUT/launches_fwd.csv python tools/profile_step.py > $OUT/ncu_launch_fwd.log 2>&1
python tools/profile_step.py --direction back > $OUT/plainb.log 2>&1 && \
ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $OUT/launches_bp.csv python tools/profile_step.py --direction back > $OUT/ncu_launch_bp.log 2>&1
ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:"k_gr_gather_strips|k_spec_gather|k_resample_window" -c 3 -o $OUT/full_fwd python tools/profile_step.py > $OUT/ncu_full_fwd.log 2>&1
ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:"k_spread_owned|k_rs_gather_strips" -c 2 -o $OUT/full_bp python tools/profile_step.py --direction back > $OUT/ncu_full_bp.log 2>&1
ls -la $OUT
