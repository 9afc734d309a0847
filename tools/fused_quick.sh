timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -2
for cfg in C2 C3 C4; do timeout 60 python tools/time_stage.py $cfg fused 3 50; done
WINO_FUSED_MERGE=2 timeout 60 python tools/time_stage.py C4 fused 3 50
timeout 120 python bench.py --no-cpu --config C4 --path fused --steps 1000 > /tmp/s.json 2>&1; python -c "
import json; d=json.load(open('/tmp/s.json')); k=d['kernels']; print('C4 fused', d['value'], d['ms_per_step'], ' '.join(f\"{n}={v['us_per_launch']}\" for n,v in k.items()))"
timeout 300 python tools/path_ab.py
