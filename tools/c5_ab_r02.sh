# C5 A/B: input-transform variant x chunk pipelines (lanes) x chunk budget
python -m pytest tests -m gpu -x -q 2>&1 | tail -2 > gpurun_out/ab_tests.txt
run() { tag=$1; shift; env "$@" > /dev/null; python bench.py --no-cpu --steps 20 $C5ARGS > gpurun_out/ab_$tag.json 2> gpurun_out/ab_$tag.err; echo "$tag $(python tools/brief_r02.py gpurun_out/ab_$tag.json | head -1 | cut -d' ' -f2-6)"; }
for v in legacy minb3; do
  if [ $v = legacy ]; then export WINO_K2F_LEGACY=1; unset WINO_K2F4_MINB; else unset WINO_K2F_LEGACY; export WINO_K2F4_MINB=3; fi
  for cfg in "0 1024" "2 256" "3 256" "3 128" "2 512"; do set -- $cfg; C5ARGS="--lanes $1 --chunk-mb $2" run ${v}_l$1_c$2; done
done
