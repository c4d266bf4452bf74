#!/bin/bash
# x-staged K1 A/B (TW_STAGE_X) + tests
mkdir -p gpurun_out; rm -f gpurun_out/stagex.log
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for rep in 1 2; do
for v in 1 0; do
  echo "== stage=$v 256" >> gpurun_out/stagex.log
  TW_STAGE_X=$v timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu-baseline --e2e-runs 1 2>&1 | tail -1 >> gpurun_out/stagex.log
  echo "== stage=$v 128" >> gpurun_out/stagex.log
  TW_STAGE_X=$v timeout 300 python bench.py --nx 128 --ny 128 --nz 128 --steps 400 --warmup 5 --no-cpu-baseline --e2e-runs 1 2>&1 | tail -1 >> gpurun_out/stagex.log
done
done
