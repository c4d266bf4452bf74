# K1 compile-time variant A/B: VARIANTS="name ..." built by
# scripts/build_variants.sh; headline iteration and event-timed K1 / K2 / K3
# at 256^3 and 128^3, alternating default / variant twice.
export PLACES=k3_pairs GRIDS=256,128
for v in default $VARIANTS default $VARIANTS; do
  if [ $v = default ]; then unset TW_HPCCG_LIB; else export TW_HPCCG_LIB=paper_2602_21897_b200/_lib/variants/libtw_hpccg_$v.so; fi
  python scripts/xupd_ab.py
done
