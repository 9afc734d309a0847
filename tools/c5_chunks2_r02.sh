# C5 (AUTO fused limit 128): chunk budget x lanes around the default (256 MiB x 3)
run() { tag=$1; shift; python bench.py --no-cpu --steps 20 "$@" > gpurun_out/cs2_$tag.json 2> gpurun_out/cs2_$tag.err; echo "$tag $(python tools/brief_r02.py gpurun_out/cs2_$tag.json | head -1 | cut -d' ' -f2-6)"; }
for cfg in "3 256" "3 384" "3 512" "2 512" "2 768" "3 192" "4 256"; do set -- $cfg; run l$1_c$2 --lanes $1 --chunk-mb $2; done
