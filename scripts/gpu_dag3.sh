#!/bin/bash
# A/B of the dispatcher's update-chunk unroll (pairs in flight per thread).
mkdir -p gpurun_out; rm -f gpurun_out/sweep_dag3.log
for lib in default u1 u3; do
  echo "== $lib" >> gpurun_out/sweep_dag3.log
  if [ $lib = default ]; then unset TW_HPCCG_LIB; else export TW_HPCCG_LIB=$PWD/paper_2602_21897_b200/_lib/variants/libtw_hpccg_$lib.so; fi
  timeout 600 python scripts/sweep.py --configs c5 --only-persistent --tiles 1,8,64,512 >> gpurun_out/sweep_dag3.log 2>&1
done
unset TW_HPCCG_LIB
timeout 600 python -m pytest tests -m gpu -q -x -k "persistent" 2>&1 | tail -2
