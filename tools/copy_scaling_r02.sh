# K3F phase scaling (debug build): copies only (WINO_FUSED_DBG=10), no MMAs (2), handshake-only epilogue (8),
# full (0) at C2 with the balanced (98 CTAs) and full (148 CTAs) grid, and copies-only vs image count.
WINO_NVCC_FLAGS=-DWINO_FUSED_DBG python -c "from paper_1901_01965_b200 import build as B; B.build(force=True)" || exit 1
for bal in 1 0; do for d in 0 2 8 10; do WINO_FUSED_BALANCE=$bal WINO_FUSED_DBG=$d python tools/time_stage.py C2 fused 3 50 | sed "s/^/bal=$bal /"; done; done
for d in 10 0; do WINO_FUSED_DBG=$d python tools/fused_scaling.py | sed "s/^/dbg=$d /"; done
python -c "from paper_1901_01965_b200 import build as B; B.build(force=True)"
