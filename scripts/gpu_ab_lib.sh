#!/bin/bash
# Same-box A/B of the monolithic CG (scripts/pdl_ab.py) between the default
# library and a variant: bash scripts/gpu_ab_lib.sh _lib/variants/<name>.so
V=paper_2602_21897_b200/$1
for rep in 1 2 3; do
  echo "== default"; timeout 300 python scripts/pdl_ab.py 2>&1 | grep graph
  echo "== $1"; TW_HPCCG_LIB=$PWD/$V timeout 300 python scripts/pdl_ab.py 2>&1 | grep graph
done
