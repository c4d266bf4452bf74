"""CPU tests of the C-ABI boundary: the product library loads without a GPU,
exports every symbol include/tw_hpccg.h declares, and fails loudly (never
silently falls back) when no B200 is present."""
import ctypes as C
import os
import subprocess

import pytest

import paper_2602_21897_b200 as P
from paper_2602_21897_b200 import _native as N


def test_library_exports_every_declared_symbol():
    lib = N.load()
    declared = N.declared_symbols()
    assert len(declared) >= 40
    missing = [s for s in declared if not hasattr(lib, s)]
    assert missing == []
    bound = {name for name, _, _ in N.SIGNATURES}
    assert set(declared) == bound, set(declared) ^ bound


def test_abi_version_and_struct_layout():
    lib = N.load()
    assert lib.tw_abi_version() == 3
    assert C.sizeof(N.EllInfo) == 13 * 8 + 2 * 4
    o = N.CgOptionsC()
    lib.tw_cg_options_default(C.byref(o))
    # CgOptions defaults (cg.hpp:37-45): tiles 16, stream pool 4, marks on, tol 0
    assert (o.variant, o.tiles, o.stream_pool_capacity, o.iteration_marks, o.tol, o.dispatch) == \
        (N.TW_CG_TASKS, 16, 4, 1, 0.0, N.TW_DISPATCH_AUTO)
    assert (o.x_update, o.l2_keep, o.dag_spmv_slices, o.dag_vec_rows) == (0, 0, 0, 0)


def test_constants_match_the_c_header():
    """Every integer constant of the header that the Python mirror binds has
    the header's value (placements, dispatch, K1 forms, transports, codes)."""
    import re
    defs = {}
    for h in N.HEADERS:
        for m in re.finditer(r"^#define\s+(TW_\w+)\s+(\d+)\b", open(h).read(), re.M):
            defs[m.group(1)] = int(m.group(2))
    for prefix in ("TW_XUPD_", "TW_L2KEEP_", "TW_DISPATCH_", "TW_K1_", "TW_TRANSPORT_", "TW_CG_",
                   "TW_ERR_"):
        names = [k for k in defs if k.startswith(prefix)]
        assert names, prefix
        for k in names:
            assert getattr(N, k) == defs[k], k
    o = P.CgOptions(x_update="k3_pairs", l2_keep=False).to_c(N.TW_CG_MONOLITHIC)
    assert (o.x_update, o.l2_keep) == (N.TW_XUPD_K3_PAIRS, N.TW_L2KEEP_OFF)
    with pytest.raises(KeyError):
        P.CgOptions(x_update="k4").to_c(N.TW_CG_MONOLITHIC)


def test_struct_layout_matches_the_c_header(tmp_path):
    """The ctypes mirrors of the ABI structs against the C compiler's own
    layout of include/tw_hpccg.h (sizeof and every field offset)."""
    structs = {"tw_cg_options": N.CgOptionsC, "tw_ell_info_t": N.EllInfo, "tw_slab_t": N.SlabPlan,
               "tw_cg_mode_t": N.CgMode}
    lines = ['#include <stddef.h>', '#include <stdio.h>', '#include "tw_hpccg.h"', "int main(void) {"]
    for cname, cls in structs.items():
        lines.append(f'printf("{cname} %zu\\n", sizeof({cname}));')
        for f, _ in cls._fields_:
            lines.append(f'printf("{cname}.{f} %zu\\n", offsetof({cname}, {f}));')
    lines.append("return 0; }")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.dirname(N.HEADER), "-o", str(exe), str(src)], check=True)
    got = dict(l.split() for l in subprocess.run([str(exe)], capture_output=True, text=True,
                                                  check=True).stdout.splitlines())
    for cname, cls in structs.items():
        assert int(got[cname]) == C.sizeof(cls), cname
        for f, _ in cls._fields_:
            assert int(got[f"{cname}.{f}"]) == getattr(cls, f).offset, (cname, f)


def test_exports_are_plain_c():
    out = subprocess.run(["nm", "-D", "--defined-only", N.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    tw = [l.split()[-1] for l in out.splitlines() if " T tw_" in l]
    assert set(N.declared_symbols()) <= set(tw)
    assert not any(s.startswith("_Z") and "tw_" in s and " T " in s for s in out.splitlines()
                   if s.split()[-1].startswith("tw_"))


def test_null_handles_are_contract_violations():
    lib = N.load()
    assert lib.tw_ctx_compute_stream(None, None) == N.TW_ERR_CONTRACT
    assert b"null" in lib.tw_last_error_string()
    assert lib.tw_cg_iterate(None, 1) == N.TW_ERR_CONTRACT
    assert lib.tw_ell_info(None, None) == N.TW_ERR_CONTRACT
    with pytest.raises(P.ContractViolation):
        N.check(lib.tw_cg_wait(None))


def test_no_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises((P.CudaError, P.ConfigError)):
        P.Runtime(0)


def test_product_package_never_imports_the_oracle():
    pkg = os.path.dirname(P.__file__)
    for root, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cpp", ".cu", ".h")):
                text = open(os.path.join(root, f)).read()
                assert "import oracle" not in text and "from oracle" not in text, f
                assert "hpccg_oracle" not in text and "libtwref" not in text, f
