#!/bin/bash
# The GPU test suite against the checked build (device bounds checks as
# traps: ELL columns / widths after every build, TMA stage bounds, halo edge
# indices, peer ranks, dispatcher task ids).  compute-sanitizer is closed
# on this pool; this is the in-kernel substitute.
set -e
cd "$(dirname "$0")/.."
# always rebuild the checked variant from the current sources
OUT=$PWD/paper_2602_21897_b200/_lib/variants/checked
make -s -C paper_2602_21897_b200/csrc -j8 OUT=$OUT NVFLAGS_EXTRA=-DTW_CHECKS >/dev/null
cp $OUT/libtw_hpccg.so paper_2602_21897_b200/_lib/variants/libtw_hpccg_checked.so
mkdir -p gpurun_out
TW_HPCCG_LIB=$PWD/paper_2602_21897_b200/_lib/variants/libtw_hpccg_checked.so \
  timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -5
TW_HPCCG_LIB=$PWD/paper_2602_21897_b200/_lib/variants/libtw_hpccg_checked.so \
  timeout 300 python scripts/sanitize_small.py 2>&1 | tail -2
