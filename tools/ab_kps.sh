for rep in 1 2; do for cfg in C3 C4; do for k in 2 4; do
  WINO_K3_KPS=$k python bench.py --no-cpu --config $cfg --path staged --steps 1000 > /tmp/s.json 2>&1; python -c "
import json; d=json.load(open('/tmp/s.json')); k=d['kernels']; print('$cfg kps $k', d['value'], d['ms_per_step'], ' '.join(f\"{n}={v['us_per_launch']}\" for n,v in k.items()))"
done; done; done
WINO_K3_KPS=4 python bench.py --no-cpu --config C5 --steps 20 > /tmp/s.json 2>&1; python -c "
import json; d=json.load(open('/tmp/s.json')); print('C5 kps4', d['value'])"
WINO_K3_KPS=2 python bench.py --no-cpu --config C5 --steps 20 > /tmp/s.json 2>&1; python -c "
import json; d=json.load(open('/tmp/s.json')); print('C5 kps2', d['value'])"
