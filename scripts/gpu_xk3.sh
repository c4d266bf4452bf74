#!/bin/bash
# x update in K3 (default) vs in K2 (TW_X_IN_K3=0), and K3 unroll variants
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
L=paper_2602_21897_b200/_lib/variants
for rep in 1 2; do
  echo "== x in K3, unroll 2 (default)"; timeout 300 python scripts/pdl_ab.py 2>&1 | grep graph
  echo "== x in K2"; TW_X_IN_K3=0 timeout 300 python scripts/pdl_ab.py 2>&1 | grep graph
  echo "== x in K3, unroll 1"; TW_HPCCG_LIB=$PWD/$L/libtw_hpccg_k3x1.so timeout 300 python scripts/pdl_ab.py 2>&1 | grep graph
  echo "== x in K3, unroll 4"; TW_HPCCG_LIB=$PWD/$L/libtw_hpccg_k3x4.so timeout 300 python scripts/pdl_ab.py 2>&1 | grep graph
done
