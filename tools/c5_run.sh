for p in auto staged; do timeout 900 python bench.py --config C5 --no-cpu --path $p > /tmp/c5_$p.json 2> /tmp/c5_$p.err; python -c "
import json; d=json.load(open('/tmp/c5_$p.json')); r=d['roofline']; print('$p', d['value'], d['ms_per_step'], d['config']['paths'], 'roof', r['kernel'], 'layer', r['layer'], r['bound'], r['frac'], 'sum/step', d['kernel_sum_vs_step'], d['clocks'])" || tail -5 /tmp/c5_$p.err; done
cp /tmp/c5_auto.json gpurun_out/pb_C5_auto.json
