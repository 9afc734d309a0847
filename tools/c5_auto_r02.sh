# C5: AUTO fused/staged threshold (WINO_AUTO_FUSED_CIN) A/B
for cin in 256 512; do WINO_AUTO_FUSED_CIN=$cin python bench.py --no-cpu --steps 20 > gpurun_out/auto_$cin.json 2> gpurun_out/auto_$cin.err; python tools/brief_r02.py gpurun_out/auto_$cin.json | sed "s/^/cin<=$cin /"; done
