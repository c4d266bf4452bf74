"""CPU check of the reference-side binding INTEGRATION.md shows: it compiles
against the reference's own headers and links against libtw_hpccg.so with
every ABI symbol resolved (no GPU needed; the reference tree is only in the
build container)."""
import os
import subprocess

import pytest

from paper_2602_21897_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_INC = "/root/reference/proj/include"


@pytest.mark.skipif(not os.path.isdir(REF_INC), reason="reference tree not present")
def test_reference_binding_compiles_and_links(tmp_path):
    src = os.path.join(ROOT, "tests", "binding", "cg_cuda_binding.cpp")
    obj, so = tmp_path / "b.o", tmp_path / "libbinding.so"
    inc = ["-I" + REF_INC, "-I" + os.path.join(ROOT, "oracle", "shim"),
           "-I" + os.path.join(ROOT, "include")]
    r = subprocess.run(["/usr/bin/g++", "-std=c++20", "-fPIC", "-c", src, "-o", str(obj)] + inc,
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]
    libdir = os.path.dirname(N.LIB_PATH)
    r = subprocess.run(["/usr/bin/g++", "-shared", "-o", str(so), str(obj), "-L" + libdir,
                        "-ltw_hpccg", "-Wl,--no-undefined", "-Wl,-rpath," + libdir],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]
    out = subprocess.run(["nm", "-D", "--undefined-only", str(so)], capture_output=True,
                         text=True).stdout
    used = {l.split()[-1] for l in out.splitlines() if l.split() and l.split()[-1].startswith("tw_")}
    assert {"tw_cg_solve", "tw_ell_from_csr", "tw_spmv_range", "tw_event_bind_async",
            "tw_stream_acquire"} <= used
