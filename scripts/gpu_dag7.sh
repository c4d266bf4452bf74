#!/bin/bash
# dispatcher tail chunks A/B (C5 256^3 and C2 128^3), same box
mkdir -p gpurun_out; rm -f gpurun_out/dag7.log
timeout 600 python -m pytest tests -m gpu -q -x -k "persistent or dispatcher or 128cubed" 2>&1 | tail -1
for rep in 1 2; do
  echo "== tail chunks (default) c5" >> gpurun_out/dag7.log
  timeout 600 python scripts/sweep.py --configs c5 --only-persistent --tiles 1,8,64,512 >> gpurun_out/dag7.log 2>&1
  echo "== no tail chunks c5" >> gpurun_out/dag7.log
  TW_DAG_SPMV_SMALL=216 TW_DAG_VEC_SMALL=32768 timeout 600 python scripts/sweep.py --configs c5 --only-persistent --tiles 1,8,64,512 >> gpurun_out/dag7.log 2>&1
done
echo "== tail chunks (default) c2" >> gpurun_out/dag7.log
timeout 600 python scripts/sweep.py --configs c2 2>&1 | grep persistent >> gpurun_out/dag7.log
echo "== no tail chunks c2" >> gpurun_out/dag7.log
TW_DAG_SPMV_SMALL=110 TW_DAG_VEC_SMALL=6912 timeout 600 python scripts/sweep.py --configs c2 2>&1 | grep persistent >> gpurun_out/dag7.log
