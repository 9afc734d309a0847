python bench.py --no-cpu --steps 300 > /tmp/s.json 2>&1; python -c "
import json; d=json.load(open('/tmp/s.json')); print('e2e', d['e2e'])"
