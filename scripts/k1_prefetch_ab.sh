# K1 L2-prefetch distance A/B (variants from scripts/build_variants.sh
# pf1="-DTW_K1_PREFETCH=1" ...): headline iteration and event-timed K1.
export PLACES=k3_pairs GRIDS=256,128
for v in default pf1 pf2 pf4 default pf1 pf2 pf4; do
  if [ $v = default ]; then unset TW_HPCCG_LIB; else export TW_HPCCG_LIB=paper_2602_21897_b200/_lib/variants/libtw_hpccg_$v.so; fi
  python scripts/xupd_ab.py
done
