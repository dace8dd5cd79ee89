"""CPU-side checks of the boundary: the C-ABI library builds, loads, exports
every entry point include/hm.h declares, and the binding declares exactly
those.  No compute call is made (no GPU here)."""
import ctypes
import os
import re

import pytest

from paper_2207_11662_b200 import build as B
from paper_2207_11662_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "hm.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:hm_status|void|const char \*)\s*\*?\s*(hm_\w+)\s*\(", src, flags=re.M)
    return sorted(set(names))


@pytest.fixture(scope="module")
def lib():
    B.build()
    return _lib.load()


def test_header_declares_expected_calls():
    names = header_functions()
    for required in ["hm_create", "hm_destroy", "hm_last_error", "hm_load_layers", "hm_and_aggregate",
                     "hm_closeness", "hm_topk_closeness", "hm_compose", "hm_free_graph", "hm_sync"]:
        assert required in names


def test_library_exports_every_declared_symbol(lib):
    for name in header_functions():
        assert hasattr(lib, name), name
        assert ctypes.cast(getattr(lib, name), ctypes.c_void_p).value


def test_binding_matches_header():
    assert sorted(_lib.SIGNATURES) == header_functions()


def test_only_abi_symbols_exported(lib):
    import subprocess
    out = subprocess.run(["nm", "-D", "--defined-only", B.LIB], capture_output=True, text=True).stdout
    syms = [ln.split()[-1] for ln in out.splitlines() if " T " in ln]
    assert syms and all(s.startswith("hm_") for s in syms), syms


def test_null_context_is_einval(lib):
    # argument checking happens before any device call
    assert lib.hm_sync(None) == _lib.HM_EINVAL
    assert lib.hm_last_error(None) == b"null context"
    assert lib.hm_create(None, 0, None) == _lib.HM_EINVAL


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2207_11662_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".c")):
                txt = open(os.path.join(dp, f)).read()
                assert "oracle" not in re.sub(r"#.*|//.*", "", txt).lower() or f == "build.py", f


def test_missing_library_fails_loudly(tmp_path):
    with pytest.raises(ImportError):
        _lib._lib = None
        try:
            _lib.load(str(tmp_path / "nope.so"))
        finally:
            _lib._lib = None
