# K3F: does the MMA work per slot-group set the pace with the epilogue running? bit 64: one UMMA per group
WINO_NVCC_FLAGS=-DWINO_FUSED_DBG python -c "from paper_1901_01965_b200 import build as B; B.build(force=True)" || exit 1
for d in 0 64 4 68 2 6; do WINO_FUSED_DBG=$d python tools/time_stage.py C2 fused 3 50; done
python -c "from paper_1901_01965_b200 import build as B; B.build(force=True)"
