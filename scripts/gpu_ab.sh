set -x
timeout 800 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
rm -f gpurun_out/ab.log
for i in 1 2; do
TW_NO_ALTERNATE=1 timeout 300 python bench.py --no-cpu-baseline --e2e-runs 1 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('fixed     ', d['value'], d['ms_per_step'], d['roofline']['avg_launch_ms'], d['roofline']['k2_update_xr_gbs'], d['roofline']['k3_update_p_gbs'])" >> gpurun_out/ab.log
timeout 300 python bench.py --no-cpu-baseline --e2e-runs 1 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('alternate ', d['value'], d['ms_per_step'], d['roofline']['avg_launch_ms'], d['roofline']['k2_update_xr_gbs'], d['roofline']['k3_update_p_gbs'])" >> gpurun_out/ab.log
done
