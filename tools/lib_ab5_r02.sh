# A/B of two library builds on one box: GPU tests (new), C5 per-layer K3F x2, C2/C3 K3F
python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for r in 1 2; do for v in new old; do
  cp paper_1901_01965_b200/libwino_$v.so paper_1901_01965_b200/libwino.so
  python bench.py --no-cpu --steps 20 > gpurun_out/ab_$v.json 2> /dev/null
  echo "$v $(python tools/brief_r02.py gpurun_out/ab_$v.json | head -1 | cut -d' ' -f2-4) | $(python -c "
import json;d=json.load(open('gpurun_out/ab_$v.json'));print(' '.join(str(round(x.get('k3_fused',0))) for x in d['layers_kernels_us'][:5]))")"
done; done
for v in new old; do cp paper_1901_01965_b200/libwino_$v.so paper_1901_01965_b200/libwino.so; python tools/time_stage.py C2 fused 3 50 | sed "s/^/$v /"; python tools/time_stage.py C3 fused 3 50 | sed "s/^/$v /"; done
cp paper_1901_01965_b200/libwino_new.so paper_1901_01965_b200/libwino.so
