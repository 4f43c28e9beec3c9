#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-r1}
# launch list of one frame (refit x2 + query) after a warm-up frame
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_${TAG}.csv python scripts/profile_query.py 2500 1500 1 > gpurun_out/launches_${TAG}.log 2>&1
# full capture of the hot kernels of the profiled frame
timeout 1500 ncu --set full --clock-control none --import-source on \
  -k regex:"k_expand|k_narrow|k_leaf_up|k_xform|k_refine" ${NCU_SKIP:---launch-skip 30} --launch-count ${NCU_COUNT:-30} \
  -o gpurun_out/prof_${TAG} -f python scripts/profile_query.py 2500 1500 1 > gpurun_out/prof_${TAG}.log 2>&1
echo "ncu exit $?" >> gpurun_out/prof_${TAG}.log
