timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "auto or vgg16" 2>&1 | tail -2
timeout 900 python bench.py --config C5 --no-cpu > /tmp/c5.json 2>/dev/null; python -c "
import json; d=json.load(open('/tmp/c5.json')); print('C5', d['value'], d['config']['paths'], d['roofline']['kernel'], d['roofline']['layer'], d['roofline']['frac'])"
