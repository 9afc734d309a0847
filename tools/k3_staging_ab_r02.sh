# staged GEMM: one output staging tile + 4 ring stages (default at c_in >= 128) vs two tiles + 3 stages, same box
for r in 1 2 3; do for v in 2 1; do
  WINO_K3_STAGING=$v python bench.py --no-cpu --steps 20 > gpurun_out/ks_$v.json 2> /dev/null
  echo "staging=$v $(python tools/brief_r02.py gpurun_out/ks_$v.json | head -1 | cut -d' ' -f2-4) | $(python -c "
import json;d=json.load(open('gpurun_out/ks_$v.json'));print(' '.join(str(round(x.get('k3_gemm',0))) for x in d['layers_kernels_us'][5:]))")"
done; done
for v in 2 1; do WINO_K3_STAGING=$v python bench.py --config C4 --no-cpu --steps 1000 > gpurun_out/ks_C4_$v.json 2>/dev/null; echo "C4 staging=$v $(python tools/brief_r02.py gpurun_out/ks_C4_$v.json | head -1 | cut -d' ' -f2-4) trials $(python -c "
import json;d=json.load(open('gpurun_out/ks_C4_$v.json'));print(d['trials']['median_tops'])")"; done
