# tests + tuning + full bench + ncu evidence, one gpurun call
set -x
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
rm -f gpurun_out/tune.log
for f in paper_2602_21897_b200/_lib/variants/*.so; do
  TW_HPCCG_LIB=$f timeout 120 python scripts/kbench.py 256 30 >> gpurun_out/tune.log 2>&1
done
timeout 120 python scripts/kbench.py 256 30 >> gpurun_out/tune.log 2>&1
timeout 120 python scripts/kbench.py 128 100 >> gpurun_out/tune.log 2>&1
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log
CMD="python bench.py --steps 6 --warmup 3 --no-cpu-baseline --e2e-runs 1"
$CMD > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:spmv_tma -s 4 -c 1 \
    -o gpurun_out/prof_k1 -f $CMD > gpurun_out/ncu_full.log 2>&1
echo "ncu exit $?"
