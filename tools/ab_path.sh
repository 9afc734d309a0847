for rep in 1 2; do for cfg in C2 C3 C4; do for path in staged fused; do
  python bench.py --no-cpu --config $cfg --path $path --steps 1000 > /tmp/s.json 2>&1; python -c "
import json; d=json.load(open('/tmp/s.json')); k=d['kernels']; print('$cfg $path', d['value'], d['ms_per_step'], d['e2e']['value'], ' '.join(f\"{n}={v['us_per_launch']}\" for n,v in k.items()))"
done; done; done
