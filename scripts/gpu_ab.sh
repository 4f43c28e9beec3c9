#!/bin/bash
# A/B of two library variants on the rings query anatomy (exp_query) plus the
# GPU tests on the default library.  VARIANTS="libgdist.so libgdist_x.so"
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
if [[ -z $NOTESTS ]]; then
  timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
  tail -3 gpurun_out/pytest_gpu.log
fi
for v in ${VARIANTS:-libgdist.so}; do
  for kind in ${KINDS:-min}; do
    echo "$v production per-frame:"; GDIST_LIB_VARIANT=$v timeout 300 python scripts/exp_frames_query.py 3 23 $kind | tail -1
  done
  [[ -n $NOANATOMY ]] && continue
  for kind in min max; do
    GDIST_LIB_VARIANT=$v timeout 300 python scripts/exp_query.py 2500 1500 7 $kind > gpurun_out/ab_${v%.so}_$kind.log 2>&1
  done
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob('gpurun_out/ab_*.log')):
    for line in open(f):
        if not line.startswith('{'):
            continue
        d = json.loads(line)
        if d['warm']: continue
        print(f, d['distance'], d['witness'], d['phases_ms'])
        print('   ', [(i['in'], i['k'], i['ms']) for i in d['iters']])
PY
for s in ${EXTRA:-}; do timeout 300 python $s > gpurun_out/$(basename $s .py).log 2>&1; cat gpurun_out/$(basename $s .py).log | tail -5; done
