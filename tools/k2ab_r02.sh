for m in 2 3 4; do WINO_K2F4_MINB=$m python tools/time_stage.py C2 fused 2 50 | sed "s/^/minb=$m /"; WINO_K2F4_MINB=$m python tools/time_stage.py C4 fused 2 50 | sed "s/^/minb=$m /"; done
WINO_K2F_LEGACY=1 python tools/time_stage.py C2 fused 2 50 | sed "s/^/legacy /"; WINO_K2F_LEGACY=1 python tools/time_stage.py C4 fused 2 50 | sed "s/^/legacy /"
