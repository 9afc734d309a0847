# HISTORICAL: the experiment switch this script exercises was removed after the measurement (not kept;
# DESIGN.md 6b records the result); kept to document how the numbers in profiles/ were taken.
# fused kernel launched as clusters of 2 / 4 CTAs (the cout blocks of a tile block co-scheduled on one GPC) vs none
WINO_FUSED_CLUSTER=4 python -m pytest tests -m gpu -x -q -k "random_shapes or lanes or full_size or c1_all" 2>&1 | tail -1
for r in 1 2; do for v in 0 2 4; do
  WINO_FUSED_CLUSTER=$v python bench.py --no-cpu --steps 20 > gpurun_out/fc_$v.json 2> gpurun_out/fc_$v.err
  echo "cluster=$v $(python tools/brief_r02.py gpurun_out/fc_$v.json | head -1 | cut -d' ' -f2-4) | $(python -c "
import json;d=json.load(open('gpurun_out/fc_$v.json'));print(' '.join(str(round(x.get('k3_fused',0))) for x in d['layers_kernels_us'][:5]))")"
done; done
for v in 0 2 4; do WINO_FUSED_CLUSTER=$v python tools/time_stage.py C2 fused 3 50 | sed "s/^/cluster=$v /"; WINO_FUSED_CLUSTER=$v python tools/time_stage.py C3 fused 3 50 | sed "s/^/cluster=$v /"; done
