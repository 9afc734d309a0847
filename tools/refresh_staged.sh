timeout 300 python bench.py --config C4 --no-cpu > gpurun_out/pb_C4.json 2>/dev/null
timeout 300 python bench.py --config C4 --path fused --no-cpu > gpurun_out/pbf_C4.json 2>/dev/null
timeout 300 python bench.py --config C3 --path staged --no-cpu > gpurun_out/pbs_C3.json 2>/dev/null
timeout 300 python bench.py --config C2 --path staged --no-cpu > gpurun_out/pbs_C2.json 2>/dev/null
timeout 900 python bench.py --config C5 --no-cpu > gpurun_out/pb_C5.json 2>/dev/null
timeout 300 python bench.py --config C3 --no-cpu > gpurun_out/pb_C3.json 2>/dev/null
timeout 300 python bench.py --config C2 > gpurun_out/pb_C2.json 2>/dev/null
for f in pb_C2 pbs_C2 pb_C3 pbs_C3 pb_C4 pbf_C4 pb_C5; do python -c "
import json; d=json.load(open('gpurun_out/$f.json')); r=d['roofline']; print('$f', d['value'], d['ms_per_step'], r['kernel'], r['bound'], r['frac'])"; done
