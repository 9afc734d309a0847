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
                       (dict(filter_target_max=127, path=1), L.WINO_ERR_UNSUPPORTED), (dict(path=3), L.WINO_ERR_INVALID_ARG),
                       (dict(algorithm=2), L.WINO_ERR_INVALID_ARG),
                       (dict(algorithm=1, path=2, input_type=1, c_in=225), L.WINO_ERR_UNSUPPORTED),
                       (dict(input_type=2), L.WINO_ERR_INVALID_ARG),
                       (dict(input_type=1, x_zero_point=256, path=2), L.WINO_ERR_INVALID_ARG),
                       (dict(input_type=1, path=1, c_in=225), L.WINO_ERR_UNSUPPORTED),
                       (dict(input_type=1, path=2, c_in=225), L.WINO_ERR_UNSUPPORTED),
                       (dict(filter_target_max=126, path=2), L.WINO_ERR_UNSUPPORTED),
                       (dict(filter_target_max=127, path=2, filter_scaling=0), L.WINO_ERR_UNSUPPORTED),
                       (dict(filter_target_max=127, path=2, algorithm=1), L.WINO_ERR_UNSUPPORTED),
                       (dict(filter_target_max=127, path=2, input_type=1), L.WINO_ERR_UNSUPPORTED),
                       (dict(lanes=9), L.WINO_ERR_INVALID_ARG), (dict(lanes=-1), L.WINO_ERR_INVALID_ARG)]:
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


def test_fast_division_matches_integer_division():
    """The kernels' tile decode divides by plan constants with a multiply-shift (layout.cuh FastDiv);
    it must equal floor division for every n in [0, 2^31) -- checked at the edges (n = q d - 1, q d,
    q d + 1, 2^31 - 1), for powers of two and their neighbours, and on random pairs."""
    import numpy as np
    import paper_1901_01965_b200._lib as L
    f = L.lib().wino_debug_fastdiv
    rng = np.random.default_rng(7)
    ds = {1, 2, 3, 5, 7, 14, 28, 49, 56, 196, 784, 3136, 12544, 2 ** 31 - 1}
    for e in range(1, 31):
        ds |= {2 ** e - 1, 2 ** e, 2 ** e + 1}
    ds |= set(int(v) for v in rng.integers(1, 2 ** 31 - 1, 200))
    top = 2 ** 31 - 1
    for d in sorted(ds):
        ns = {0, 1, d - 1, d, d + 1, top, top - 1, top - d, (top // d) * d, (top // d) * d - 1}
        ns |= set(int(v) for v in rng.integers(0, top, 20))
        for q in (1, 2, 3, 1000):
            ns |= {q * d - 1, q * d, q * d + 1}
        for n in ns:
            if 0 <= n <= top:
                assert f(n, d) == n // d, (n, d)
    assert f(-1, 3) == -1 and f(5, 0) == -1


def test_bench_reports_uint8_above_its_cin_limit_as_unsupported():
    """bench.py --input u8 on a config whose c_in exceeds the uint8 limit (A28: 224) prints one JSON line that
    says so (no CUDA needed: the check precedes any launch) instead of failing inside wino_plan."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--config", "C4", "--input", "u8", "--no-cpu"],
                       capture_output=True, text=True, timeout=300, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert "unsupported" in line and "224" in line["unsupported"]
