#!/bin/bash
# dispatcher chunk-size defaults at 128^3 and 256^3, same box
mkdir -p gpurun_out; rm -f gpurun_out/dag5.log
timeout 600 python -m pytest tests -m gpu -q -x -k "persistent or dispatcher or 128cubed" 2>&1 | tail -1
for cfg in "default" "55/3542" "55/8192" "108/3328"; do
  echo "== c2 $cfg" >> gpurun_out/dag5.log
  if [ $cfg = default ]; then unset TW_DAG_SPMV_SLICES TW_DAG_VEC_ROWS; else
    export TW_DAG_SPMV_SLICES=${cfg%/*} TW_DAG_VEC_ROWS=${cfg#*/}; fi
  timeout 600 python scripts/sweep.py --configs c2 2>&1 | grep persistent >> gpurun_out/dag5.log
done
unset TW_DAG_SPMV_SLICES TW_DAG_VEC_ROWS
echo "== c5 default" >> gpurun_out/dag5.log
timeout 600 python scripts/sweep.py --configs c5 --only-persistent --tiles 1,8,64,512 >> gpurun_out/dag5.log 2>&1
