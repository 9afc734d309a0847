WINO_K3_PAIR=1 timeout 300 python -m pytest tests -m gpu -x -q -k "staged or STAGED or auto or full_size" 2>&1 | tail -2
bash tools/k3_pair2_r02.sh
