# The round's evidence in one gpurun call: GPU tests, smoke, bench (default
# and long), the reference arm, the ncu launch list and --set full captures
# of K1 / K2 / K3 (each ncu pass only after its command ran clean without
# ncu); then, here: python scripts/summarize_ncu.py gpurun_out/launches.csv
# gpurun_out/prof_k1.ncu-rep <round tag>
set -x
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log
timeout 600 python bench.py --steps 600 --warmup 10 --no-cpu-baseline --no-extras --e2e-runs 1 > gpurun_out/bench_long.log 2>&1; echo "bench exit $?" >> gpurun_out/bench_long.log
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "bench exit $?" >> gpurun_out/bench_ref.log
CMD="python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-extras --e2e-runs 1"
$CMD > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:spmv_tma -s 4 -c 1 \
    -o gpurun_out/prof_k1 -f $CMD > gpurun_out/ncu_full.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:update_xr -s 4 -c 1 \
    -o gpurun_out/prof_k2 -f $CMD > gpurun_out/ncu_full_k2.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:update_p_kernel<.*0, .*0>" -s 2 -c 1 \
    -o gpurun_out/prof_k3 -f $CMD > gpurun_out/ncu_full_k3.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:update_p_kernel<.*0, .*2>" -s 2 -c 1 \
    -o gpurun_out/prof_k3p -f $CMD > gpurun_out/ncu_full_k3p.log 2>&1
echo "ncu exit $?"
