CMD="python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-extras --e2e-runs 1"
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:update_p_kernel<.*0, .*0>" -s 2 -c 1 \
    -o gpurun_out/prof_k3 -f $CMD > gpurun_out/ncu_full_k3.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:update_p_kernel<.*0, .*2>" -s 2 -c 1 \
    -o gpurun_out/prof_k3p -f $CMD > gpurun_out/ncu_full_k3p.log 2>&1
echo "ncu exit $?"
