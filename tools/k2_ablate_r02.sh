WINO_NVCC_FLAGS=-DWINO_K2_DBG python -c "from paper_1901_01965_b200 import build as B; B.build(force=True)" || exit 1
for n in 32 128 512; do for d in 0 1 2 3; do WINO_K2_DBG=$d python tools/k2_ablate_r02.py $n; done; done
python -c "from paper_1901_01965_b200 import build as B; B.build(force=True)"
