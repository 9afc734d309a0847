# Round-1 profile refresh: bench lines (default auto path and the other path), the reference arm,
# ncu launch lists and --set full captures for both kernel paths at C2.
set -x
python bench.py --config C2 > gpurun_out/pb_C2.json 2> gpurun_out/pb_C2.err
python bench.py --config C2 --path staged --no-cpu > gpurun_out/pbs_C2.json 2> gpurun_out/pbs_C2.err
for c in C3 C4 C5; do timeout 600 python bench.py --config $c --no-cpu > gpurun_out/pb_$c.json 2> gpurun_out/pb_$c.err; done
timeout 300 python bench.py --config C3 --path staged --no-cpu > gpurun_out/pbs_C3.json 2> gpurun_out/pbs_C3.err
timeout 300 python bench.py --config C4 --path fused --no-cpu > gpurun_out/pbf_C4.json 2> gpurun_out/pbf_C4.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/pref_C2.json 2> gpurun_out/pref_C2.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_C2.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_launch.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_C2_staged.csv python bench.py --steps 2 --warmup 3 --no-cpu --path staged >> gpurun_out/ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -c 4 -o gpurun_out/full_C2_fused python tools/run_conv.py C2 fused 1 > gpurun_out/ncu_full.log 2>&1
ncu --set full --import-source on --clock-control none -c 4 -o gpurun_out/full_C2 python tools/run_conv.py C2 staged 1 >> gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out | tail -30
