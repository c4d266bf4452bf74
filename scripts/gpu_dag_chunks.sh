#!/bin/bash
# chunk-size sweep of the 19-warp x 1-CTA dispatcher (C5 256^3, C2 128^3) + dispatcher tests
mkdir -p gpurun_out; rm -f gpurun_out/sweep_dag5.log
timeout 600 python -m pytest tests -m gpu -q -x -k "persistent or dispatcher or 128cubed" 2>&1 | tail -2
for cfg in "default default" "108 32768" "432 32768" "864 32768" "216 65536" "216 16384"; do
  set -- $cfg
  echo "== spmv_slices=$1 vec_rows=$2" >> gpurun_out/sweep_dag5.log
  if [ "$1" = default ]; then
    timeout 600 python scripts/sweep.py --configs c5,c2 --only-persistent --tiles 4,16,64 >> gpurun_out/sweep_dag5.log 2>&1
  else
    TW_DAG_SPMV_SLICES=$1 TW_DAG_VEC_ROWS=$2 timeout 600 python scripts/sweep.py --configs c5,c2 --only-persistent --tiles 4,16,64 >> gpurun_out/sweep_dag5.log 2>&1
  fi
done
