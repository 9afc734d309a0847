# C5 staged layers: K3 K-steps per stage x ring depth cap (sensitivity of the copy-latency-bound GEMM)
run() { tag=$1; shift; env "$@" python bench.py --no-cpu --steps 20 > gpurun_out/kr_$tag.json 2> gpurun_out/kr_$tag.err; echo "$tag $(python tools/brief_r02.py gpurun_out/kr_$tag.json | head -2 | tr '\n' ' ' | cut -c1-90) | $(python -c "
import json;d=json.load(open('gpurun_out/kr_$tag.json'));print(' '.join(str(round(x.get('k3_gemm',0))) for x in d['layers_kernels_us'][5:]))")"; }
run base X=0
run kps2 WINO_K3_KPS=2
run kps2_st5 WINO_K3_KPS=2 WINO_K3_STAGES=5
run kps2_st4 WINO_K3_KPS=2 WINO_K3_STAGES=4
run kps4_st2 WINO_K3_KPS=4 WINO_K3_STAGES=2
