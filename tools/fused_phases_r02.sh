# K3F phase ablation (debug build): bit 2 no MMAs, 4 no copies, 8 handshake-only epilogue; C2 and C3
WINO_NVCC_FLAGS=-DWINO_FUSED_DBG python -c "from paper_1901_01965_b200 import build as B; B.build(force=True)" || exit 1
for c in C2 C3; do for d in 0 2 4 6 8 10 12 14; do WINO_FUSED_DBG=$d python tools/time_stage.py $c fused 3 50; done; done
python -c "from paper_1901_01965_b200 import build as B; B.build(force=True)"
