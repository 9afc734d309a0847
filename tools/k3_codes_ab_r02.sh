# staged GEMM after dropping the shared-memory code table: the default rule (one staging tile at c_in >= 512)
# vs always two, same box; plus the GPU tests
python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for r in 1 2; do for v in 0 2; do
  WINO_K3_STAGING=$v python bench.py --no-cpu --steps 20 > gpurun_out/kc_$v.json 2> /dev/null
  echo "staging=$v $(python tools/brief_r02.py gpurun_out/kc_$v.json | head -1 | cut -d' ' -f2-4) | $(python -c "
import json;d=json.load(open('gpurun_out/kc_$v.json'));print(' '.join(str(round(x.get('k3_gemm',0))) for x in d['layers_kernels_us'][5:]))")"
done; done
