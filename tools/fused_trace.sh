WINO_NVCC_FLAGS="-DWINO_FUSED_TRACE" python -c "from paper_1901_01965_b200 import build as B; B.build(force=True)"
timeout 120 python tools/trace_fused.py C2 0 | tail -62
python -c "from paper_1901_01965_b200 import build as B; B.build(force=True)"
