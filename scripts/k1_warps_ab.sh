export PLACES=k3_pairs GRIDS=256,128
for v in default w19 w20 w16 default w19 w20; do
  if [ $v = default ]; then unset TW_HPCCG_LIB; else export TW_HPCCG_LIB=paper_2602_21897_b200/_lib/variants/libtw_hpccg_$v.so; fi
  python scripts/xupd_ab.py
  python -c "
import paper_2602_21897_b200 as P
rt=P.Runtime(0); A=P.gen_stencil_matrix(256,256,256,rt=rt); S=P.CgSolver(rt,A,5,P.CgOptions(tiles=1),variant=0); print('$v mode', S.mode()['k1_kernel'])"
done
