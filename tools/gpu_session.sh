#!/bin/bash
# Full profiling session on the GPU box with the summaries made there, so that
# only text comes back (the .ncu-rep captures exceed gpurun's 64 MiB limit):
#   gpurun -- 'bash tools/gpu_session.sh r2z'
TAG=${1:-r2z}
bash tools/gpu_profile.sh $TAG > gpurun_out/${TAG}_session.log 2>&1
bash tools/gpu_profile_c4.sh ${TAG}_c4 >> gpurun_out/${TAG}_session.log 2>&1
python tools/summarize_profiles.py $TAG >> gpurun_out/${TAG}_session.log 2>&1
python tools/summarize_profiles.py ${TAG}_c4 >> gpurun_out/${TAG}_session.log 2>&1
mkdir -p gpurun_out/${TAG}_profiles
cp profiles/${TAG}_* gpurun_out/${TAG}_profiles/
cp gpurun_out/$TAG/*.err gpurun_out/${TAG}_profiles/ 2>/dev/null
rm -rf gpurun_out/$TAG gpurun_out/${TAG}_c4
ls -la gpurun_out/${TAG}_profiles
