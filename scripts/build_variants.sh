# Build compile-time variants of libtw_hpccg.so into _lib/variants/ (tuning
# A/Bs; the product is the default build).  Each argument is NAME=FLAGS, e.g.
#   bash scripts/build_variants.sh k2rev="-DTW_K2_REV=1 -DTW_K2_KEEP_R=1"
set -e
cd "$(dirname "$0")/../paper_2602_21897_b200/csrc"
OUT=../_lib/variants; mkdir -p $OUT
for cfg in "$@"; do
  NAME=${cfg%%=*}; FLAGS=${cfg#*=}
  d=$(mktemp -d)
  make -s -C . OUT=$d NVFLAGS_EXTRA="$FLAGS" >/dev/null 2>&1
  cp $d/libtw_hpccg.so $OUT/libtw_hpccg_$NAME.so; rm -rf $d
done
ls $OUT
