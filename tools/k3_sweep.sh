for cfg in C2 C4; do for bal in 0 1; do
  WINO_K3_BALANCE=$bal python bench.py --no-cpu --config $cfg --path staged --steps 1000 > /tmp/s.json 2>&1; python -c "
import json; d=json.load(open('/tmp/s.json')); k=d['kernels']; print('$cfg bal $bal', d['value'], d['ms_per_step'], ' '.join(f\"{n}={v['us_per_launch']}\" for n,v in k.items()))"
done; done
for cfg in C2 C3; do python bench.py --no-cpu --config $cfg --steps 1000 > /tmp/s.json 2>&1; python -c "
import json; d=json.load(open('/tmp/s.json')); k=d['kernels']; print('$cfg default', d['value'], d['ms_per_step'], ' '.join(f\"{n}={v['us_per_launch']}\" for n,v in k.items()))"; done
