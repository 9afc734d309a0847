# K3 bottleneck probe (debug build with -DWINO_K3_DBG; the normal build is restored afterwards):
# stage-3 launch time under the WINO_K3_DBG ablation modes
WINO_NVCC_FLAGS=-DWINO_K3_DBG python -c "from paper_1901_01965_b200 import build as B; B.build(force=True)"
for cfg in C2 C4; do
  for d in 0 1 2 4 8 6 10 12 14; do
    WINO_K3_DBG=$d python tools/time_stage.py $cfg staged 3 50 | sed "s/^/dbg=$d /"
  done
done
python -c "from paper_1901_01965_b200 import build as B; B.build(force=True)"
