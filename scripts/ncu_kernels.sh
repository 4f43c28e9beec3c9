#!/bin/bash
# full ncu capture of the query kernels of one rings frame (after a warm-up
# frame): k_traverse, k_seed, k_narrow, k_refine [+ refit kernels]
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-r1}
KIND=${KIND:-min}
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:"${KREGEX:-k_traverse|k_narrow|k_refine|k_seed|k_leaf_up|k_xform}" --launch-skip ${SKIP:-6} --launch-count ${COUNT:-8} \
  -o gpurun_out/prof_${TAG} -f python scripts/profile_query.py 2500 1500 1 ${KIND} > gpurun_out/prof_${TAG}.log 2>&1
echo "ncu exit $?" >> gpurun_out/prof_${TAG}.log
