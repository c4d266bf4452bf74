# Same-box A/B of the monolithic CG between the default library and the
# variants built into _lib/variants/ (scripts/build_variants.sh), alternating;
# SM clocks and throttle reasons logged before each run.
V=paper_2602_21897_b200/_lib/variants
clk() { nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,clocks_throttle_reasons.active --format=csv,noheader; }
for rep in 1 2; do
  echo "clocks: $(clk)"; timeout 300 python scripts/iter_ab.py
  for f in $V/*.so; do echo "clocks: $(clk)"; TW_HPCCG_LIB=$PWD/$f timeout 300 python scripts/iter_ab.py; done
done
