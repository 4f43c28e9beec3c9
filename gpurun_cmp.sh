cd /root/repo
for k in min max min max; do
  timeout 120 python scripts/exp_query.py 2500 1500 7 $k 2>&1 | python -c "
import json,sys
for line in sys.stdin:
    if not line.startswith('{'): continue
    d=json.loads(line)
    if d['warm']: continue
    print('$k', d['phases_ms'], d['distance'])
"
done
timeout 400 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -1
