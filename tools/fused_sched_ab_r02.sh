# HISTORICAL: the experiment switch this script exercises was removed after the measurement (not kept;
# DESIGN.md 6b records the result); kept to document how the numbers in profiles/ were taken.
# fused-kernel unit schedule: strided (default) vs contiguous ranges per CTA (WINO_FUSED_SCHED=1), same box
WINO_FUSED_SCHED=1 python -m pytest tests -m gpu -x -q -k "random_shapes or lanes or c1_all or full_size_configs" 2>&1 | tail -1
for r in 1 2; do for v in 0 1; do
  WINO_FUSED_SCHED=$v python bench.py --no-cpu --steps 20 > gpurun_out/fs_$v.json 2> /dev/null
  echo "sched=$v $(python tools/brief_r02.py gpurun_out/fs_$v.json | head -1 | cut -d' ' -f2-4) | $(python -c "
import json;d=json.load(open('gpurun_out/fs_$v.json'));print(' '.join(str(round(x.get('k3_fused',0))) for x in d['layers_kernels_us'][:5]))")"
done; done
for c in C2 C3; do for v in 0 1; do WINO_FUSED_SCHED=$v python tools/time_stage.py $c fused 3 50 | sed "s/^/sched=$v /"; done; done
