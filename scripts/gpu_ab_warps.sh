L=$PWD/paper_2602_21897_b200/_lib/variants
for r in 1 2; do
  echo "== default (18 warps)"; timeout 300 python scripts/k23_times.py 2>&1 | grep 256
  for v in w16s1 w17s1 w19s1; do echo "== $v"; TW_HPCCG_LIB=$L/libtw_hpccg_$v.so timeout 300 python scripts/k23_times.py 2>&1 | grep 256; done
done
