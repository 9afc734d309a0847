# CTA-pair staged GEMM (WINO_K3_PAIR=1): parity first (bounded by timeouts), then C4 stage times and C5 lines
export WINO_K3_PAIR=1
timeout 300 python -m pytest tests -m gpu -x -q -k "staged or STAGED or path2 or auto or full_size" 2>&1 | tail -5
echo "pytest rc=$?"
timeout 120 python tools/time_stage.py C4 staged 3 50 | sed "s/^/pair /"
WINO_K3_PAIR=0 timeout 120 python tools/time_stage.py C4 staged 3 50 | sed "s/^/base /"
for v in 1 0; do WINO_K3_PAIR=$v timeout 300 python bench.py --no-cpu --steps 20 > gpurun_out/kp_$v.json 2> gpurun_out/kp_$v.err; echo "pair=$v $(python tools/brief_r02.py gpurun_out/kp_$v.json | head -1 | cut -d' ' -f2-4) | $(python -c "
import json;d=json.load(open('gpurun_out/kp_$v.json'));print(' '.join(str(round(x.get('k3_gemm',0))) for x in d['layers_kernels_us'][5:]))" 2>&1 | tail -1)"; done
