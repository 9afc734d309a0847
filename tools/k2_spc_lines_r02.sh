# K2F slices per CTA: C2-C4 bench lines at spc 1 and 4 (default), then the GPU tests at the default
for c in C2 C3 C4; do for v in 1 4; do WINO_K2F4_SPC=$v python bench.py --config $c --no-cpu --steps 1000 > gpurun_out/sl_${c}_$v.json 2>/dev/null; echo "$c spc=$v $(python tools/brief_r02.py gpurun_out/sl_${c}_$v.json | head -1 | cut -d' ' -f2-4)"; done; done
python -m pytest tests -m gpu -x -q 2>&1 | tail -1
