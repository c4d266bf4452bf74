#!/bin/bash
# dispatcher CTA width A/B (warps per CTA incl. the scheduler warp), C5 256^3
mkdir -p gpurun_out; rm -f gpurun_out/dagw.log
for lib in dag17x1 dag19x1 dag21x1; do
  if [ $lib = default ]; then unset TW_HPCCG_LIB; else export TW_HPCCG_LIB=$PWD/paper_2602_21897_b200/_lib/variants/libtw_hpccg_$lib.so; fi
  echo "== $lib" >> gpurun_out/dagw.log
  timeout 600 python scripts/sweep.py --configs c5 --only-persistent --tiles 1,8,64,512 >> gpurun_out/dagw.log 2>&1
done
