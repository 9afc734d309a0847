# A/B of the K1 carveout preference, interleaved repeats (C2, C3, C4)
for rep in 1 2 3; do for cfg in C2 C3 C4; do for co in 0 25 -1; do
  WINO_CARVE_K1=$co python bench.py --no-cpu --config $cfg --steps 1000 > /tmp/s.json 2>&1; python -c "
import json; d=json.load(open('/tmp/s.json')); k=d['kernels']; print('$cfg carve $co', d['value'], d['ms_per_step'], ' '.join(f\"{n}={v['us_per_launch']}\" for n,v in k.items()))"
done; done; done
