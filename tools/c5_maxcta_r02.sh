# C5: cap on the fused kernel's grid (the other lanes' K2 run on the freed SMs) x lanes
run() { tag=$1; shift; env "$@" python bench.py --no-cpu --steps 20 $ARGS > gpurun_out/mc_$tag.json 2> gpurun_out/mc_$tag.err; echo "$tag $(python tools/brief_r02.py gpurun_out/mc_$tag.json | head -1 | cut -d' ' -f2-6)"; }
python -m pytest tests -m gpu -q -x -k "write_only" 2>&1 | tail -1
for c in 0 136 124 112 100; do ARGS="" run cap$c WINO_FUSED_MAXCTA=$c; done
for c in 0 124; do ARGS="--lanes 4" run l4_cap$c WINO_FUSED_MAXCTA=$c; done
