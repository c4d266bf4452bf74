set -x
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 -k "persistent" > gpurun_out/pytest_dag.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_dag.log
rm -f gpurun_out/sweep_dag.log
for cfg in "16 4096" "32 4096" "16 8192" "8 2048" "48 16384"; do
  set -- $cfg
  echo "== spmv_slices=$1 vec_rows=$2" >> gpurun_out/sweep_dag.log
  TW_DAG_SPMV_SLICES=$1 TW_DAG_VEC_ROWS=$2 timeout 600 python scripts/sweep.py --configs c5 --only-persistent --tiles 1,8,64,512 >> gpurun_out/sweep_dag.log 2>&1
done
