#!/bin/bash
# tile-kernel grid share A/B for the tasks variant (streams + graph), C2 and C5
mkdir -p gpurun_out; rm -f gpurun_out/tilegrid.log
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
for mode in share full; do
  if [ $mode = full ]; then export TW_TILE_GRID=full; else unset TW_TILE_GRID; fi
  echo "== $mode c2" >> gpurun_out/tilegrid.log
  timeout 600 python scripts/sweep.py --configs c2 2>&1 | grep -v persistent >> gpurun_out/tilegrid.log
  echo "== $mode c5" >> gpurun_out/tilegrid.log
  timeout 900 python scripts/sweep.py --configs c5 --tiles 1,4,16,64,256 2>&1 | grep -v persistent >> gpurun_out/tilegrid.log
done
