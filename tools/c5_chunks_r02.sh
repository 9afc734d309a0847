# C5 sweep: chunk pipelines (lanes) x chunk budget (MiB), small budgets keep a chunk's V resident in L2
run() { tag=$1; shift; python bench.py --no-cpu --steps 20 "$@" > gpurun_out/cs_$tag.json 2> gpurun_out/cs_$tag.err; echo "$tag $(python tools/brief_r02.py gpurun_out/cs_$tag.json | head -1 | cut -d' ' -f2-6)"; }
for l in 1 2 3; do for c in 16 32 64 256; do run l${l}_c$c --lanes $l --chunk-mb $c; done; done
