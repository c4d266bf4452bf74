set -x
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 -k "persistent" > gpurun_out/pytest_dag.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_dag.log
rm -f gpurun_out/sweep_dag.log
for f in default paper_2602_21897_b200/_lib/dagvariants/*.so; do
  echo "== $f" >> gpurun_out/sweep_dag.log
  if [ $f = default ]; then L=""; else L="TW_HPCCG_LIB=$f"; fi
  env $L timeout 600 python scripts/sweep.py --configs c5 --only-persistent --tiles 1,8,64,512 >> gpurun_out/sweep_dag.log 2>&1
done
