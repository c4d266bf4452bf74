#!/bin/bash
# peer-instantiation K3 unroll A/B (1-rank communicator, 256^3)
mkdir -p gpurun_out; rm -f gpurun_out/pk3.log
for lib in default pu2 pu3; do
  if [ $lib = default ]; then unset TW_HPCCG_LIB; else export TW_HPCCG_LIB=$PWD/paper_2602_21897_b200/_lib/variants/libtw_hpccg_$lib.so; fi
  for i in 1 2; do
    echo "== $lib" >> gpurun_out/pk3.log
    timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu-baseline --e2e-runs 1 --comm 2>&1 | tail -1 >> gpurun_out/pk3.log
  done
done
