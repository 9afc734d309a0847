# K3F per-CTA timeline at C2 (trace build): full kernel and the no-copy / no-MMA ablations
WINO_NVCC_FLAGS="-DWINO_FUSED_TRACE -DWINO_FUSED_DBG" python -c "from paper_1901_01965_b200 import build as B; B.build(force=True)" || exit 1
for d in 0 4 2; do echo "== dbg $d"; WINO_FUSED_DBG=$d timeout 120 python tools/trace_fused.py C2 0; done
python -c "from paper_1901_01965_b200 import build as B; B.build(force=True)"
