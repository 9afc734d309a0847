# C5: K2F resident CTAs per SM (register budget) 2 / 3 (default) / 4
for m in 3 4 2; do WINO_K2F4_MINB=$m python bench.py --no-cpu --steps 20 > gpurun_out/km_$m.json 2> gpurun_out/km_$m.err; echo "minb $m: $(python tools/brief_r02.py gpurun_out/km_$m.json | head -2 | tr '\n' ' ' | cut -c1-600)"; done
