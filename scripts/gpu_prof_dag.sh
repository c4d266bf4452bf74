#!/bin/bash
# ncu --set full of the persistent DAG dispatcher (C5 256^3, 64 tiles) and,
# for comparison, of the monolithic K1 in the same sweep process.
mkdir -p gpurun_out
timeout 300 python scripts/sweep.py --configs c5 --only-persistent --tiles 64 --K 3 --W 1 > gpurun_out/dag_prof_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dag_kernel -c 1 \
  -o gpurun_out/prof_dag -f python scripts/sweep.py --configs c5 --only-persistent --tiles 64 --K 3 --W 1 \
  > gpurun_out/ncu_dag.log 2>&1; echo "ncu exit $?"
