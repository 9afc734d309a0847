timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -2
for cfg in C2 C3 C4; do timeout 60 python tools/time_stage.py $cfg fused 3 50; done
for cfg in C2 C3; do timeout 120 python bench.py --no-cpu --config $cfg --steps 1000 > /tmp/s.json 2>&1; python -c "
import json; d=json.load(open('/tmp/s.json')); k=d['kernels']; print('$cfg', d['value'], d['ms_per_step'], d['config']['path'], ' '.join(f\"{n}={v['us_per_launch']}\" for n,v in k.items()))"; done
