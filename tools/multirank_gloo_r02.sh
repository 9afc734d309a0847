# the multi-rank bench flow on real kernels (gloo validation mode: ranks share the one GPU; no data-path
# collective, so their kernels never wait on one another; timings are not per-GPU numbers)
export WINO_DIST_BACKEND=gloo
timeout 600 python bench.py --gpus 2 --config C2 --steps 50 --no-cpu > gpurun_out/mr_C2x2.json 2> gpurun_out/mr_C2x2.err; echo "C2 x2 rc=$?"
timeout 600 python bench.py --gpus 8 --config C1 --steps 50 --no-cpu > gpurun_out/mr_C1x8.json 2> gpurun_out/mr_C1x8.err; echo "C1 x8 rc=$?"
timeout 900 python bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu > gpurun_out/mr_C5x2.json 2> gpurun_out/mr_C5x2.err; echo "C5 x2 rc=$?"
for f in mr_C2x2 mr_C1x8 mr_C5x2; do python -c "
import json,sys
l=[x for x in open('gpurun_out/$f.json') if x.startswith('{')]
d=json.loads(l[-1]) if l else {}
print('$f', d.get('n_gpus'), d.get('value'), d.get('config',{}).get('parallelism'), json.dumps(d.get('sharded_check')), json.dumps(d.get('self_check'))[:160])
"; tail -3 gpurun_out/$f.err; done
