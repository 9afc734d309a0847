# K3F epilogue ablation (debug build): bit 128 = no reverse-scale multiply (an add instead), 8 = handshake only;
# C5 layers 1-2 conv times and C2 K3F
WINO_NVCC_FLAGS=-DWINO_FUSED_DBG python -c "from paper_1901_01965_b200 import build as B; B.build(force=True)" > /dev/null 2>&1 || exit 1
for d in 0 128 8 2 130; do
  echo "== dbg $d" >> gpurun_out/epi.txt
  WINO_FUSED_DBG=$d python tools/c5_layers_r02.py 2>&1 | grep "layer  [1-3]:" | cut -c1-60 >> gpurun_out/epi.txt
  WINO_FUSED_DBG=$d python tools/time_stage.py C2 fused 3 50 >> gpurun_out/epi.txt 2>&1
done
python -c "from paper_1901_01965_b200 import build as B; B.build(force=True)" > /dev/null 2>&1
