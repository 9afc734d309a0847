# CTA-pair staged GEMM: ring shapes (K steps per stage 2 / 4 / 8) vs the single-CTA kernel, C4 stage time
for k in 4 8; do WINO_K3_PAIR=1 WINO_K3_KPS=$k timeout 120 python tools/time_stage.py C4 staged 3 50 | sed "s/^/pair kps=$k /"; done
WINO_K3_PAIR=0 timeout 120 python tools/time_stage.py C4 staged 3 50 | sed "s/^/base /"
for k in 4; do WINO_K3_PAIR=1 WINO_K3_KPS=$k timeout 120 python tools/time_stage.py C3 staged 3 50 | sed "s/^/pair C3 kps=$k /"; done
WINO_K3_PAIR=0 timeout 120 python tools/time_stage.py C3 staged 3 50 | sed "s/^/base C3 /"
