# refresh every committed bench line of round 1 (default AUTO lines with the reference and CPU baseline at C2)
set -x
timeout 600 python bench.py --config C2 > gpurun_out/pb_C2.json 2> gpurun_out/pb_C2.err
timeout 300 python bench.py --config C2 --path staged --no-cpu > gpurun_out/pbs_C2.json 2>/dev/null
timeout 300 python bench.py --config C3 --no-cpu > gpurun_out/pb_C3.json 2>/dev/null
timeout 300 python bench.py --config C3 --path staged --no-cpu > gpurun_out/pbs_C3.json 2>/dev/null
timeout 300 python bench.py --config C4 --no-cpu > gpurun_out/pb_C4.json 2>/dev/null
timeout 300 python bench.py --config C4 --path staged --no-cpu > gpurun_out/pbs_C4.json 2>/dev/null
timeout 900 python bench.py --config C5 --no-cpu > gpurun_out/pb_C5.json 2>/dev/null
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/pref_C2.json 2>/dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_C2.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_launch.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_C2_staged.csv python bench.py --steps 2 --warmup 3 --no-cpu --path staged >> gpurun_out/ncu_launch.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -c 4 -o gpurun_out/full_C2_fused python tools/run_conv.py C2 fused 1 > gpurun_out/ncu_full.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -c 4 -o gpurun_out/full_C2 python tools/run_conv.py C2 staged 1 >> gpurun_out/ncu_full.log 2>&1
for f in pb_C2 pbs_C2 pb_C3 pbs_C3 pb_C4 pbs_C4 pb_C5; do python -c "
import json; d=json.load(open('gpurun_out/$f.json')); r=d['roofline']; print('$f', d['value'], d['ms_per_step'], r['kernel'], r['bound'], r['frac'], d['e2e']['value'])"; done
