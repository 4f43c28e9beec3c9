#!/bin/bash
# Round-2 evidence pass (one gpurun call): launch list of one rings frame,
# ncu --set full of every kernel of the second frame (min and max queries,
# NVTX range "frame1"), and compute-sanitizer memcheck / racecheck /
# synccheck on desk-scale queries (grid barrier, refit cascade, exact pass).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-r2a}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_${TAG}.csv python scripts/profile_query.py 2500 1500 1 > gpurun_out/launches_${TAG}.log 2>&1
for KIND in min max; do
  timeout 1200 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "frame1/" \
    -o gpurun_out/prof_${TAG}_${KIND} -f python scripts/profile_query.py 2500 1500 1 ${KIND} \
    > gpurun_out/prof_${TAG}_${KIND}.log 2>&1
  echo "ncu exit $?" >> gpurun_out/prof_${TAG}_${KIND}.log
done
# the refit kernel of one frame (both trees), ncu --set full
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_refit --launch-skip 4 --launch-count 2 \
  -o gpurun_out/prof_${TAG}_refit -f python scripts/exp_refit.py > gpurun_out/prof_${TAG}_refit.log 2>&1
echo "ncu exit $?" >> gpurun_out/prof_${TAG}_refit.log
if [[ -z "$NO_SANITIZER" ]]; then
  for TOOL in memcheck racecheck synccheck; do
    timeout 900 compute-sanitizer --tool ${TOOL} --print-limit 20 --error-exitcode 9 \
      python scripts/sanitize_desk.py > gpurun_out/sanitizer_${TOOL}.log 2>&1
    echo "compute-sanitizer ${TOOL} exit $?" >> gpurun_out/sanitizer_${TOOL}.log
  done
fi
