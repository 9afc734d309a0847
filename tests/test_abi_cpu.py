"""CPU-side checks of the boundary: the C-ABI library builds, loads and exports
every symbol include/wino.h declares; argument validation that happens
before any CUDA call.  No compute calls (no GPU here)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_symbols():
    txt = open(os.path.join(ROOT, "include", "wino.h")).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(wino_\w+)\s*\(", txt, re.M)))


def test_library_builds_and_exports_every_header_symbol():
    from paper_1901_01965_b200 import build as B
    B.build()
    L = ctypes.CDLL(B.LIB)
    syms = _header_symbols()
    assert len(syms) >= 13
    for s in syms:
        assert hasattr(L, s), s
    import paper_1901_01965_b200._lib as PL
    assert sorted(PL.EXPORTS) == syms


def test_status_strings_and_pre_cuda_validation():
    import paper_1901_01965_b200._lib as L
    assert L.status_string(0) == "ok"
    assert "unsupported" in L.status_string(L.WINO_ERR_UNSUPPORTED)
    base = dict(n=1, h=8, w=8, c_in=4, c_out=4, pad=1, layout=1, filter_scaling=1, filter_target_max=255,
                out_mode=0)
    for kw, status in [(dict(pad=2), L.WINO_ERR_UNSUPPORTED), (dict(c_in=897, filter_scaling=0), L.WINO_ERR_UNSUPPORTED),
                       (dict(c_in=769), L.WINO_ERR_UNSUPPORTED), (dict(layout=5), L.WINO_ERR_INVALID_ARG),
                       (dict(out_mode=9), L.WINO_ERR_INVALID_ARG), (dict(h=1, pad=0), L.WINO_ERR_UNSUPPORTED),
                       (dict(filter_target_max=127), L.WINO_ERR_UNSUPPORTED), (dict(path=3), L.WINO_ERR_INVALID_ARG),
                       (dict(algorithm=2), L.WINO_ERR_INVALID_ARG),
                       (dict(algorithm=1, path=1, input_type=1, c_in=225), L.WINO_ERR_UNSUPPORTED),
                       (dict(input_type=2), L.WINO_ERR_INVALID_ARG),
                       (dict(input_type=1, x_zero_point=256, path=1), L.WINO_ERR_INVALID_ARG),
                       (dict(input_type=1, path=0, c_in=225), L.WINO_ERR_UNSUPPORTED),
                       (dict(input_type=1, path=1, c_in=225), L.WINO_ERR_UNSUPPORTED),
                       (dict(filter_target_max=126, path=1), L.WINO_ERR_UNSUPPORTED),
                       (dict(filter_target_max=127, path=1, filter_scaling=0), L.WINO_ERR_UNSUPPORTED),
                       (dict(filter_target_max=127, path=1, algorithm=1), L.WINO_ERR_UNSUPPORTED),
                       (dict(filter_target_max=127, path=1, input_type=1), L.WINO_ERR_UNSUPPORTED)]:
        d = dict(base); d.update(kw)
        with pytest.raises(L.WinoError) as e:
            L.wino_plan(L.wino_conv_desc(**d), 0)
        assert e.value.status == status, kw


def test_sizes_of_null_plan_are_zero():
    import paper_1901_01965_b200._lib as L
    assert L.wino_filter_bytes(None) == 0 and L.wino_workspace_bytes(None) == 0


def test_product_package_does_not_import_oracle():
    """The product path never touches oracle/ (no CPU fallback)."""
    pkg = os.path.join(ROOT, "paper_1901_01965_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"(import\s+oracle|from\s+oracle|liboracle|oracle\.c\b|oracle/)", txt), f
