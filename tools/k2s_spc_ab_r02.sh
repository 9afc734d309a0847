# staged / F(2x2) / legacy-fused K2 with slices per CTA 1 vs 4 (default): GPU tests, C4 staged K2, C5
python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for v in 1 4; do
  WINO_K2_SPC=$v python tools/time_stage.py C4 staged 2 50 | sed "s/^/spc=$v /"
  WINO_K2_SPC=$v python tools/time_stage.py C2 staged 2 50 | sed "s/^/spc=$v /"
done
for r in 1 2; do for v in 1 4; do
  WINO_K2_SPC=$v python bench.py --no-cpu --steps 20 > gpurun_out/s2_$v.json 2> /dev/null
  echo "spc=$v $(python tools/brief_r02.py gpurun_out/s2_$v.json | head -1 | cut -d' ' -f2-4) | $(python -c "
import json;d=json.load(open('gpurun_out/s2_$v.json'));print(' '.join(str(round(x.get('k2_input',0))) for x in d['layers_kernels_us'][5:]))")"
done; done
