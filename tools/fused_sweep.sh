for cfg in C2 C3; do for bal in 0 1; do for st in 2 3 4; do
  WINO_FUSED_BALANCE=$bal python bench.py --no-cpu --config $cfg --streams $st --steps 1000 > /tmp/s.json 2>&1; python -c "
import json; d=json.load(open('/tmp/s.json')); k=d['kernels']; print('$cfg bal $bal streams $st', d['value'], d['ms_per_step'], ' '.join(f\"{n}={v['us_per_launch']}\" for n,v in k.items()))"
done; done; done
