# K3 timeline (debug build with -DWINO_K3_TRACE; the normal build is restored afterwards)
WINO_NVCC_FLAGS=-DWINO_K3_TRACE python -c "from paper_1901_01965_b200 import build as B; B.build(force=True)"
python tools/trace_gemm.py C2
WINO_K3_DBG=14 python tools/trace_gemm.py C2
WINO_K3_DBG=2 python tools/trace_gemm.py C2
python -c "from paper_1901_01965_b200 import build as B; B.build(force=True)"
