#!/bin/bash
# A/B of the K3->K1 fusion (TW_FUSE_P) at 256^3 and 128^3 plus the GPU tests.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for sz in 256 128; do
  st=250; [ $sz = 128 ] && st=500
  for f in 1 0; do
    TW_FUSE_P=$f timeout 300 python bench.py --nx $sz --ny $sz --nz $sz --steps $st --warmup 5 \
      --no-cpu-baseline > gpurun_out/bf${f}_$sz.json 2>&1 || echo "bench fuse=$f $sz failed"
  done
done
