# K3F: is the MMA slowed by the epilogue's TMEM traffic? bits 16 no re-zeroing, 32 no accumulator loads
WINO_NVCC_FLAGS=-DWINO_FUSED_DBG python -c "from paper_1901_01965_b200 import build as B; B.build(force=True)" || exit 1
for d in 0 16 32 48 4 20 36 52 12; do WINO_FUSED_DBG=$d python tools/time_stage.py C2 fused 3 50; done
python -c "from paper_1901_01965_b200 import build as B; B.build(force=True)"
