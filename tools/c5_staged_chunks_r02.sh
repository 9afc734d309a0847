# HISTORICAL: the experiment switch this script exercises was removed after the measurement (not kept;
# DESIGN.md 6b records the result); kept to document how the numbers in profiles/ were taken.
# C5: chunk budget / lanes of the staged layers only (M'' + V per chunk small enough to stay in L2)
run() { tag=$1; shift; env "$@" python bench.py --no-cpu --steps 20 > gpurun_out/sc_$tag.json 2> gpurun_out/sc_$tag.err; echo "$tag $(python tools/brief_r02.py gpurun_out/sc_$tag.json | head -1 | cut -d' ' -f2-4) | $(python -c "
import json;d=json.load(open('gpurun_out/sc_$tag.json'));print(' '.join(str(round(sum(x.values()))) for x in d['layers_kernels_us'][5:]), d['config']['chunks'][5:])")"; }
run base X=0
run s64_l1 WINO_STACK_STAGED_MB=64 WINO_STACK_STAGED_LANES=1
run s96_l1 WINO_STACK_STAGED_MB=96 WINO_STACK_STAGED_LANES=1
run s48_l2 WINO_STACK_STAGED_MB=48 WINO_STACK_STAGED_LANES=2
run s128_l2 WINO_STACK_STAGED_MB=128 WINO_STACK_STAGED_LANES=2
run base2 X=0
