#!/bin/bash
# K3 unroll A/B (single-domain and 1-rank peer), 256^3
mkdir -p gpurun_out; rm -f gpurun_out/k3ab.log
for lib in default k3u4; do
  if [ $lib = default ]; then unset TW_HPCCG_LIB; else export TW_HPCCG_LIB=$PWD/paper_2602_21897_b200/_lib/variants/libtw_hpccg_$lib.so; fi
  for i in 1 2; do
    echo "== $lib single" >> gpurun_out/k3ab.log
    timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu-baseline --e2e-runs 1 >> gpurun_out/k3ab.log 2>&1
    echo "== $lib peer1" >> gpurun_out/k3ab.log
    timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu-baseline --e2e-runs 1 --comm >> gpurun_out/k3ab.log 2>&1
  done
done
unset TW_HPCCG_LIB
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
