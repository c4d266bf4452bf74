#!/bin/bash
# dispatcher update chunks: full GPU suite, then update-chunk size A/B (TMA blocks)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for v in default 16384 65536; do
  echo "== TW_DAG_VEC_ROWS=$v"
  if [ $v = default ]; then unset TW_DAG_VEC_ROWS; else export TW_DAG_VEC_ROWS=$v; fi
  timeout 600 python scripts/sweep.py --configs c5 --only-persistent --tiles 1,4,8,16,64,512 2>&1 | \
    python3 -c "import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l)
        if d.get('dispatch')=='persistent': print(d['config'][:3], d['tiles'], round(d['ms_per_iter'],4))"
done
unset TW_DAG_VEC_ROWS
timeout 600 python scripts/sweep.py --configs c5,c2 --tiles 1,2,4,8,16,32,64,128,256,512 > gpurun_out/sweep_final.jsonl 2>&1
