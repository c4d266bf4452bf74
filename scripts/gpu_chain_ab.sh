# Same-box A/B of the programmatic chain (scripts/chain_ab.py, CHAIN_ONLY) and
# of the monolithic CG (scripts/iter_ab.py) between the default library and
# the variants built into _lib/variants/ (scripts/build_variants.sh).
V=paper_2602_21897_b200/_lib/variants
for rep in 1 2; do
  CHAIN_ONLY=1 timeout 600 python scripts/chain_ab.py
  [ -n "$MONO" ] && timeout 300 python scripts/iter_ab.py
  for f in $V/*.so; do
    CHAIN_ONLY=1 TW_HPCCG_LIB=$PWD/$f timeout 600 python scripts/chain_ab.py
    [ -n "$MONO" ] && TW_HPCCG_LIB=$PWD/$f timeout 300 python scripts/iter_ab.py
  done
done
