# Build TMA SpMV tuning variants (warps per CTA x stages per warp) into _lib/variants/
set -e
cd "$(dirname "$0")/../paper_2602_21897_b200/csrc"
OUT=../_lib/variants; mkdir -p $OUT
for cfg in "$@"; do
  W=${cfg%x*}; S=${cfg#*x}
  d=$(mktemp -d)
  make -s -C . OUT=$d NVFLAGS_EXTRA="-DTW_TMA_WARPS=$W -DTW_TMA_STAGES=$S" >/dev/null
  cp $d/libtw_hpccg.so $OUT/libtw_hpccg_w${W}s${S}.so; rm -rf $d
done
ls $OUT
