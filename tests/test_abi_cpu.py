"""Boundary checks that need no GPU: the C-ABI library loads and exports every
symbol include/vrs.h declares; the header and the binding agree; no compute
call is made here."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "vrs.h")


def _declared():
    src = open(HDR).read()
    return sorted(set(re.findall(r"VRS_API\s+[\w\s\*]+?\b(vrs_\w+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = _declared()
    for must in ("vrs_load", "vrs_search", "vrs_select", "vrs_merge", "vrs_free", "vrs_last_error"):
        assert must in names


def test_library_loads_and_exports_every_declared_symbol():
    import paper_2403_15807_b200 as vrs
    lib = vrs.library()
    for name in _declared():
        assert hasattr(lib, name), f"libvrs.so does not export {name}"
    assert set(_declared()) == set(vrs.EXPORTS)


def test_header_constants_match_binding():
    import paper_2403_15807_b200._lib as L
    src = open(HDR).read()
    assert int(re.search(r"#define VRS_K_MAX (\d+)", src).group(1)) == L.K_MAX
    assert int(re.search(r"#define VRS_MAX_CLAUSES (\d+)", src).group(1)) == L.MAX_CLAUSES
    for name, val in (("VRS_EINVAL", L.EINVAL), ("VRS_ENOTFOUND", L.ENOTFOUND), ("VRS_EDEGENERATE", L.EDEGENERATE),
                      ("VRS_EUNSUPPORTED", L.EUNSUPPORTED), ("VRS_COSINE", L.COSINE), ("VRS_PATH_GEMM", L.PATH_GEMM),
                      ("VRS_ROWS_MASKED", L.ROWS_MASKED)):
        assert int(re.search(name + r"\s*=\s*(\d+)", src).group(1)) == val


def test_library_is_sm100a_only():
    so = os.path.join(ROOT, "paper_2403_15807_b200", "libvrs.so")
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out.replace("sm_100a", ""))


def test_product_never_references_oracle():
    pkg = os.path.join(ROOT, "paper_2403_15807_b200")
    for dp, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dp, f), errors="replace").read()
                assert "import oracle" not in txt and "from oracle" not in txt and "vrs_oracle" not in txt, f


def test_missing_library_fails_loudly(tmp_path, monkeypatch):
    import paper_2403_15807_b200._lib as L
    monkeypatch.setattr(L, "LIB_PATH", str(tmp_path / "nope.so"))
    monkeypatch.setattr(L, "_lib", None)
    with pytest.raises(ImportError):
        L.load_library()


def test_product_library_exports_exactly_the_header():
    """libvrs.so's dynamic symbol table is the boundary and nothing else: no debug-only
    entry points (e.g. the -DVRS_TC_TIMING timeline reader) and no leaked internals."""
    import subprocess
    so = os.path.join(ROOT, "paper_2403_15807_b200", "libvrs.so")
    out = subprocess.run(["nm", "-D", "--defined-only", so], capture_output=True, text=True, check=True).stdout
    exported = sorted(line.split()[-1] for line in out.splitlines() if line.strip())
    assert exported == _declared()
