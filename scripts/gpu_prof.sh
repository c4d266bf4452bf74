# ncu evidence for the bench command (run only after the same command exits 0)
set -x
CMD="python bench.py --steps 6 --warmup 3 --no-cpu-baseline --e2e-runs 1"
$CMD > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:spmv_kernel -s 4 -c 1 \
    -o gpurun_out/prof_k1 -f $CMD > gpurun_out/ncu_full.log 2>&1
echo "exit $?"
