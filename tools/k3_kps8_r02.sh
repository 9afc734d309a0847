# staged GEMM: 8 K steps per 96 KB stage (two stages, one staging tile) vs the default, same box
WINO_K3_KPS=8 python -m pytest tests -m gpu -x -q -k "random_shapes or full_size or max_cin or lanes" 2>&1 | tail -1
for r in 1 2; do for v in 0 8; do
  WINO_K3_KPS=$v python bench.py --no-cpu --steps 20 > gpurun_out/k8_$v.json 2> /dev/null
  echo "kps=$v $(python tools/brief_r02.py gpurun_out/k8_$v.json | head -1 | cut -d' ' -f2-4) | $(python -c "
import json;d=json.load(open('gpurun_out/k8_$v.json'));print(' '.join(str(round(x.get('k3_gemm',0))) for x in d['layers_kernels_us'][5:]))")"
done; done
for v in 0 8; do WINO_K3_KPS=$v python tools/time_stage.py C4 staged 3 50 | sed "s/^/kps=$v /"; done
