WINO_NVCC_FLAGS="-DWINO_FUSED_TRACE -DWINO_FUSED_DBG" python -c "from paper_1901_01965_b200 import build as B; B.build(force=True)"
python tools/trace_fused.py C2 0
WINO_FUSED_DBG=10 python tools/trace_fused.py C2 0
python -c "from paper_1901_01965_b200 import build as B; B.build(force=True)"
