# ncu --set full of one K1 launch (bench.py's 5th) of the default build and,
# with VARIANT=name, of _lib/variants/libtw_hpccg_<name>.so too
CMD="python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-extras --e2e-runs 1"
ncu --set full --clock-control none --import-source on -k regex:spmv_tma -s 4 -c 1 \
    -o gpurun_out/prof_k1_default -f $CMD > gpurun_out/ncu_k1_default.log 2>&1
if [ -n "$VARIANT" ]; then
  TW_HPCCG_LIB=paper_2602_21897_b200/_lib/variants/libtw_hpccg_$VARIANT.so \
  ncu --set full --clock-control none --import-source on -k regex:spmv_tma -s 4 -c 1 \
      -o gpurun_out/prof_k1_$VARIANT -f $CMD > gpurun_out/ncu_k1_$VARIANT.log 2>&1
fi
echo "ncu exit $?"
