# refresh the SURVEY 8(f) variant bench lines (staged path)
for c in C2 C3 C4; do timeout 300 python bench.py --config $c --alg f2 --path staged --no-cpu > gpurun_out/v_${c}_f2.json 2>/dev/null; done
for c in C2 C3; do timeout 300 python bench.py --config $c --input u8 --path staged --no-cpu > gpurun_out/v_${c}_u8.json 2>/dev/null; done
for c in C2 C3; do timeout 300 python bench.py --config $c --target 127 --path staged --no-cpu > gpurun_out/v_${c}_f3.json 2>/dev/null; done
for f in gpurun_out/v_*.json; do python -c "
import json; d=json.load(open('$f')); print('$f', d['value'], d['ms_per_step'], d['config']['path'], d['scaling_error']['out32_lsb'] if d.get('scaling_error') else None)"; done
