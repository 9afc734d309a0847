# K3F debug ablation: bit 256 = no epilogue shared-memory traffic (Z_0/Z_5 parking, staging, output stores);
# with and without MMAs (bit 2); C2 and C5 layers 1-3
WINO_NVCC_FLAGS=-DWINO_FUSED_DBG python -c "from paper_1901_01965_b200 import build as B; B.build(force=True)" > /dev/null 2>&1 || exit 1
for d in 0 8192 4096 2048; do
  echo "== dbg $d" >> gpurun_out/es.txt
  WINO_FUSED_DBG=$d python tools/time_stage.py C2 fused 3 50 >> gpurun_out/es.txt 2>&1
  WINO_FUSED_DBG=$d python tools/c5_layers_r02.py 2>&1 | grep "layer  [1-3]:" | cut -c1-60 >> gpurun_out/es.txt
done
python -c "from paper_1901_01965_b200 import build as B; B.build(force=True)" > /dev/null 2>&1
