"""The C-ABI library builds, loads, exports every symbol include/usp.h
declares, and rejects bad arguments with a status (no GPU needed: no
compute call is made)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "usp.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(usp_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2207_14222_b200 import build as B

    B.build()
    from paper_2207_14222_b200 import _lib

    return _lib.load()


def test_every_declared_symbol_is_exported(lib):
    syms = declared_symbols()
    assert len(syms) >= 17
    for s in syms:
        assert hasattr(lib, s), s
    from paper_2207_14222_b200 import _lib

    assert set(syms) == set(_lib.SIGNATURES), "binding must cover exactly the header"


def test_version_and_error_strings(lib):
    assert lib.usp_version().startswith(b"0.4")
    assert isinstance(lib.usp_last_error(), bytes)


def test_argument_errors_return_status(lib):
    from paper_2207_14222_b200 import _lib

    h = ctypes.c_void_p()
    assert lib.usp_plan_create(None, ctypes.byref(h)) == 1            # USP_ERR_ARG
    d = _lib.PlanDesc()
    d.ndim = 0
    assert lib.usp_plan_create(ctypes.byref(d), ctypes.byref(h)) == 1
    d.ndim, d.D = 2, 1.0
    d.n[0], d.n[1] = 48, 64                                           # 48: not a power of two
    d.h[0] = d.h[1] = 1.0
    assert lib.usp_plan_create(ctypes.byref(d), ctypes.byref(h)) == 5  # USP_ERR_UNSUPPORTED
    assert b"power of two" in lib.usp_last_error()
    d.n[0] = 4096
    assert lib.usp_plan_create(ctypes.byref(d), ctypes.byref(h)) == 5
    d.n[0], d.D = 64, -1.0
    assert lib.usp_plan_create(ctypes.byref(d), ctypes.byref(h)) == 1
    lib.usp_plan_destroy(None)                                        # no-op


def test_product_does_not_touch_oracle():
    """The CUDA product and the oracle share no code and neither imports the
    other."""
    pkg = os.path.join(ROOT, "paper_2207_14222_b200")
    bad_prod = re.compile(r"^\s*(from\s+oracle|import\s+oracle|#\s*include\s+\"[^\"]*oracle)", re.M)
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f), errors="replace").read()
                assert not bad_prod.search(txt), f
    bad_orc = re.compile(r"^\s*(from\s+paper_2207_14222_b200|import\s+paper_2207_14222_b200|#\s*include\s+\"[^\"]*(usp\.h|fft_core|kernels))", re.M)
    for f in os.listdir(os.path.join(ROOT, "oracle")):
        if f.endswith((".py", ".c", ".h")):
            assert not bad_orc.search(open(os.path.join(ROOT, "oracle", f)).read()), f


def test_no_environment_switches_in_the_product():
    """What a plan computes is chosen by usp_plan_desc fields, not by the
    environment: the only getenv in the library is the NCCL path hint."""
    csrc = os.path.join(ROOT, "paper_2207_14222_b200", "csrc")
    hits = []
    for f in sorted(os.listdir(csrc)):
        txt = open(os.path.join(csrc, f), errors="replace").read()
        hits += [(f, m) for m in re.findall(r"getenv\(\s*\"([A-Z0-9_]+)\"", txt)]
    assert hits == [("usp_api.cu", "USP_NCCL_LIB")], hits


def test_desc_binding_matches_header():
    """The ctypes PlanDesc mirrors usp_plan_desc field by field."""
    from paper_2207_14222_b200 import _lib

    src = open(os.path.join(ROOT, "include", "usp.h")).read()
    body = src[src.index("typedef struct {\n    int ndim;"):src.index("} usp_plan_desc;")]
    body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
    names = re.findall(r"\b([A-Za-z_0-9]+)(?:\[\d\])?;", body)
    assert names == [f[0] for f in _lib.PlanDesc._fields_]


C_CLIENT = r"""
#include <stdio.h>
#include <string.h>
#include "usp.h"
int main(void) {
    usp_plan_desc d;
    memset(&d, 0, sizeof d);
    d.ndim = 3; d.n[0] = 64; d.n[1] = 64; d.n[2] = 100;   /* 100: not a power of two */
    d.h[0] = d.h[1] = d.h[2] = 1.0; d.D = 1.0;
    usp_plan_t p = 0;
    usp_status s = usp_plan_create(&d, &p);
    char msg[512];
    strncpy(msg, usp_last_error(), sizeof msg - 1);
    msg[sizeof msg - 1] = 0;
    int kind = -1;
    usp_status s2 = usp_transport(0, &kind);                /* NULL plan: an error status */
    printf("%s|%d|%d|%s\n", usp_version(), (int)s, (int)s2, msg);
    return (s == USP_ERR_UNSUPPORTED && p == 0 && s2 == USP_ERR_ARG) ? 0 : 1;
}
"""


def test_plain_c_client(lib, tmp_path):
    """The boundary is C: include/usp.h compiles as C99 and a C program
    linked against libusp.so gets validation errors as statuses (no GPU)."""
    import shutil
    import subprocess

    gcc = shutil.which("gcc")
    if gcc is None:
        pytest.skip("gcc not available")
    src = tmp_path / "client.c"
    src.write_text(C_CLIENT)
    exe = tmp_path / "client"
    libdir = os.path.join(ROOT, "paper_2207_14222_b200")
    subprocess.run([gcc, "-std=c99", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), str(src), "-L", libdir,
                    "-lusp", "-Wl,-rpath," + libdir, "-o", str(exe)], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    version, status, status2, msg = r.stdout.strip().split("|", 3)
    assert version.startswith("0.4") and int(status) == 5 and int(status2) == 1 and "power of two" in msg
