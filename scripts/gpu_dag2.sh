#!/bin/bash
# Persistent dispatcher chunk-size sweep, larger chunks (C5 256^3, 1 B200).
mkdir -p gpurun_out
rm -f gpurun_out/sweep_dag2.log
for cfg in "48 16384" "96 16384" "96 32768" "144 32768" "192 65536"; do
  set -- $cfg
  echo "== spmv_slices=$1 vec_rows=$2" >> gpurun_out/sweep_dag2.log
  TW_DAG_SPMV_SLICES=$1 TW_DAG_VEC_ROWS=$2 timeout 600 python scripts/sweep.py --configs c5 --only-persistent --tiles 1,8,64,512 >> gpurun_out/sweep_dag2.log 2>&1
done
