# fused stage variants on C5's fused layers: WINO_FUSED_MERGE 4 (default) vs 1 (MG 2/3 off: layers 4-5 general ring)
for r in 1 2; do for v in 4 1; do
  WINO_FUSED_MERGE=$v python bench.py --no-cpu --steps 20 > gpurun_out/fm_$v.json 2> /dev/null
  echo "merge=$v $(python tools/brief_r02.py gpurun_out/fm_$v.json | head -1 | cut -d' ' -f2-4) | $(python -c "
import json;d=json.load(open('gpurun_out/fm_$v.json'));print(' '.join(str(round(x.get('k3_fused',0))) for x in d['layers_kernels_us'][:5]))")"
done; done
