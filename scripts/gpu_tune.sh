set -x
timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
rm -f gpurun_out/tune.log
for f in paper_2602_21897_b200/_lib/variants/*.so; do
  TW_HPCCG_LIB=$f timeout 120 python scripts/kbench.py 256 30 >> gpurun_out/tune.log 2>&1
done
timeout 120 python scripts/kbench.py 256 30 >> gpurun_out/tune.log 2>&1
