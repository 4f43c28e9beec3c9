#!/bin/bash
# quick GPU iteration: gpu tests + per-iteration anatomy of min & max rings queries
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python scripts/exp_query.py 2500 1500 7 min > gpurun_out/exp_min.log 2>&1
timeout 300 python scripts/exp_query.py 2500 1500 7 max > gpurun_out/exp_max.log 2>&1
python - <<'PY'
import json
for f in ['gpurun_out/exp_min.log', 'gpurun_out/exp_max.log']:
    for line in open(f):
        if not line.startswith('{'):
            print(line.rstrip()); continue
        d = json.loads(line)
        if d['warm']: continue
        print(d['distance'], d['witness'], d['phases_ms'], 'narrow_pairs', d['narrow_pairs'])
        print('   ', [(i['in'], i['ms'], i['sweep_ms']) for i in d['iters']])
PY
