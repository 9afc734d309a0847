WINO_NVCC_FLAGS="-DWINO_FUSED_TRACE -DWINO_FUSED_DBG" python -c "from paper_1901_01965_b200 import build as B; B.build(force=True)"
echo "== full"; timeout 120 python tools/trace_fused.py C2 0 | sed -n '2,20p'
echo "== no UMMAs"; WINO_FUSED_DBG=2 timeout 120 python tools/trace_fused.py C2 0 | sed -n '2,20p'
python -c "from paper_1901_01965_b200 import build as B; B.build(force=True)"
