# K2F: 16-channel slices per CTA (1 = default, 2, 4: the warps reading the same pixels share L1), same box
WINO_K2F4_SPC=4 python -m pytest tests -m gpu -x -q -k "random_shapes or lanes or c1_all or full_size_configs or extremes" 2>&1 | tail -1
for v in 1 2 4; do
  for c in C2 C4; do WINO_K2F4_SPC=$v python tools/time_stage.py $c fused 2 50 | sed "s/^/spc=$v /"; done
  WINO_K2F4_SPC=$v python tools/k2_ablate_r02.py 512 | sed "s/^/spc=$v /"
done
for r in 1 2; do for v in 1 4; do
  WINO_K2F4_SPC=$v python bench.py --no-cpu --steps 20 > gpurun_out/sp_$v.json 2> /dev/null
  echo "spc=$v $(python tools/brief_r02.py gpurun_out/sp_$v.json | head -1 | cut -d' ' -f2-4) | $(python -c "
import json;d=json.load(open('gpurun_out/sp_$v.json'));print(' '.join(str(round(x.get('k2_input',0))) for x in d['layers_kernels_us'][:5]))")"
done; done
