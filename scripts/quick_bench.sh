#!/bin/bash
# Usage (GPU box): bash scripts/quick_bench.sh cfg2 cfg5 ...  -> one summary line per workload
for w in "$@"; do
  python bench.py --workload $w --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); s=d.get('steps_ms') or {}
print(d['config']['workload'][:5], '%.4g tuples/s' % d['value'], 'ms/step %.4f' % d['ms_per_step'],
      's1a %.4f s1b %.4f s2b %.4f' % (s.get('s1a_delta_dict',0), s.get('s1b_dict_merge',0), s.get('s2b_recompress',0)),
      'frac', (d.get('roofline') or {}).get('frac'))"
done
