#!/bin/bash
# Config-4 (100M-point NUFFT) session: launch list + ncu full of gather/spread -> gpurun_out/$TAG
TAG=${1:-c4}
OUT=gpurun_out/$TAG
mkdir -p $OUT
P="python tools/profile_step.py --config 4"
$P > $OUT/plain.log 2>&1 && \
ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $OUT/launches.csv $P > $OUT/ncu_launch.log 2>&1 && \
ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:"k_spread_owned|k_gather_binned" -c 2 -o $OUT/full $P > $OUT/ncu_full.log 2>&1
ls -la $OUT
