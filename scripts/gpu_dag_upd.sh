#!/bin/bash
# GPU suite, then the dispatcher / tasks sweep with the x update in the p-update chunks
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for v in 1 0; do
  echo "== TW_X_IN_K3=$v"
  TW_X_IN_K3=$v timeout 600 python scripts/sweep.py --configs c5 --tiles 1,4,16,64,512 2>&1 | \
    python3 -c "import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l)
        m='persistent' if d.get('dispatch')=='persistent' else ('graph' if d.get('cuda_graph') else 'streams')
        print(d['config'][:3], d.get('tiles'), m, round(d['ms_per_iter'],4))"
done
