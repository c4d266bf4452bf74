#!/bin/bash
# dispatcher chunk sizes at 128^3
mkdir -p gpurun_out; rm -f gpurun_out/dag6.log
for cfg in "55/8192" "108/8192" "108/16384" "216/8192" "110/6912"; do
  echo "== c2 $cfg" >> gpurun_out/dag6.log
  export TW_DAG_SPMV_SLICES=${cfg%/*} TW_DAG_VEC_ROWS=${cfg#*/}
  timeout 600 python scripts/sweep.py --configs c2 2>&1 | grep persistent >> gpurun_out/dag6.log
done
