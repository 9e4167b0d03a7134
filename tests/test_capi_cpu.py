"""CPU-side checks of the native boundary: the in-tree library builds for
sm_100a, loads without a GPU, and exports every symbol include/nimbus_cop.h
declares; the binding's signature table covers the same set; and no product
module imports the oracle."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "nimbus_cop.h")


def header_functions():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(nimbus_[a-z0-9_]+)\s*\(", txt)))


@pytest.fixture(scope="module")
def built():
    import __graft_entry__ as g
    g.build()
    from paper_2411_15707_b200 import nimbus
    return nimbus


def test_header_declares_the_boundary():
    fns = header_functions()
    for must in ("nimbus_ctx_create", "nimbus_keygen", "nimbus_encrypt_weights", "nimbus_cop_matmul",
                 "nimbus_decrypt", "nimbus_cop_matmul_host"):
        assert must in fns


def test_library_exports_every_header_symbol(built):
    lib = ctypes.CDLL(built.LIB_PATH)
    missing = [f for f in header_functions() if not hasattr(lib, f)]
    assert not missing, missing
    assert sorted(built.EXPORTED) == header_functions()


def test_library_is_sm100a_with_tcgen05(built):
    out = subprocess.run(["cuobjdump", "-sass", built.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in subprocess.run(["cuobjdump", "-lelf", built.LIB_PATH], capture_output=True,
                                       text=True).stdout
    assert "UTCIMMA" in out        # tcgen05.mma kind::i8
    assert "UBLKCP" in out         # bulk async copies into shared memory
    assert "LDTM" in out           # tcgen05.ld from tensor memory


def test_no_cpu_fallback_without_library(tmp_path, monkeypatch):
    from paper_2411_15707_b200 import nimbus
    monkeypatch.setattr(nimbus, "LIB_PATH", str(tmp_path / "missing.so"))
    monkeypatch.setattr(nimbus, "_lib", None)
    with pytest.raises(ImportError):
        nimbus.lib()


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2411_15707_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dp, f)).read()
                assert "oracle" not in re.sub(r"(#|//).*", "", txt).lower().replace("oracle/", ""), f
