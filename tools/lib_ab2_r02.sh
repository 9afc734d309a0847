# A/B of two library builds on one box: C5 lines (with SM clocks) x3 each, then the new build's GPU tests
for r in 1 2 3; do for v in new old; do
  cp paper_1901_01965_b200/libwino_$v.so paper_1901_01965_b200/libwino.so
  python bench.py --no-cpu --steps 30 > gpurun_out/ab_$v.json 2> /dev/null
  echo "$v $(python tools/brief_r02.py gpurun_out/ab_$v.json | head -1 | cut -d' ' -f2-4) clk $(python -c "
import json;d=json.load(open('gpurun_out/ab_$v.json'));print(d['clocks']['sm_mhz'], d['clocks']['reasons'], d['trials']['median_tops'])")"
done; done
cp paper_1901_01965_b200/libwino_new.so paper_1901_01965_b200/libwino.so
python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for v in new old; do cp paper_1901_01965_b200/libwino_$v.so paper_1901_01965_b200/libwino.so; python tools/time_stage.py C2 fused 3 50 | sed "s/^/$v /"; python tools/time_stage.py C4 staged 3 50 | sed "s/^/$v /"; done
cp paper_1901_01965_b200/libwino_new.so paper_1901_01965_b200/libwino.so
