for rep in 1 2 3; do for p in fused staged; do timeout 200 python bench.py --no-cpu --config C4 --path $p --steps 1000 > /tmp/s.json 2>&1; python -c "
import json; d=json.load(open('/tmp/s.json')); k=d['kernels']; print('C4 $p', d['value'], d['ms_per_step'])"; done; done
for cin in 128 256; do WINO_AUTO_FUSED_CIN=$cin timeout 600 python bench.py --no-cpu --config C5 --steps 10 > /tmp/c5.json 2>&1; python -c "
import json; d=json.load(open('/tmp/c5.json')); print('C5 auto<=$cin', d['value'], d['config']['paths'])"; done
