# Same-box A/B of the programmatic chain (scripts/chain_ab.py, CHAIN_ONLY) between
# the default library and variants built into _lib/variants/.
V=paper_2602_21897_b200/_lib/variants
for rep in 1 2; do
  CHAIN_ONLY=1 timeout 600 python scripts/chain_ab.py
  CHAIN_ONLY=1 TW_HPCCG_LIB=$PWD/$V/libtw_hpccg_lateexit.so timeout 600 python scripts/chain_ab.py
done
