set -x
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 -k "persistent" > gpurun_out/pytest_dag.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_dag.log
timeout 900 python scripts/sweep.py --configs c5,c2 > gpurun_out/sweep_dag.log 2>&1; echo "sweep exit $?" >> gpurun_out/sweep_dag.log
