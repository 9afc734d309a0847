# L2-residency sweep: chunk budget (V + M'' per chunk) x streams in flight, C2 and C4
for cfg in C2 C4; do
for st in 1 2 3; do
  for mb in 128 64 48 32; do
    WINO_CHUNK_MB=$mb python bench.py --config $cfg --steps 300 --warmup 5 --no-cpu --streams $st > /tmp/b.json 2>/dev/null
    python -c "
import json; d=json.load(open('/tmp/b.json'))
k=d['kernels']; print('$cfg streams=$st chunkMB=$mb chunks', d['config']['chunks'], 'TOPS', d['value'], 'ms', d['ms_per_step'], ' '.join(f\"{n}={v['us_per_launch']}x{v['launches_per_step']}\" for n,v in k.items()))"
  done
done
done
