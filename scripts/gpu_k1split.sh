#!/bin/bash
# K1 split column/value pipeline A/B (256^3, 128^3) + GPU tests
mkdir -p gpurun_out; rm -f gpurun_out/k1ab.log
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for rep in 1 2; do
for lib in default k1old; do
  if [ $lib = default ]; then unset TW_HPCCG_LIB; else export TW_HPCCG_LIB=$PWD/paper_2602_21897_b200/_lib/variants/libtw_hpccg_$lib.so; fi
  echo "== $lib 256" >> gpurun_out/k1ab.log
  timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu-baseline --e2e-runs 1 >> gpurun_out/k1ab.log 2>&1
  echo "== $lib 128" >> gpurun_out/k1ab.log
  timeout 300 python bench.py --nx 128 --ny 128 --nz 128 --steps 400 --warmup 5 --no-cpu-baseline --e2e-runs 1 >> gpurun_out/k1ab.log 2>&1
done
done
