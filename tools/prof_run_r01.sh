set -x
python bench.py --config C2 > gpurun_out/pb_C2.json 2> gpurun_out/pb_C2.err
for c in C3 C4 C5; do timeout 600 python bench.py --config $c --no-cpu > gpurun_out/pb_$c.json 2> gpurun_out/pb_$c.err; done
for c in C2 C3 C4; do timeout 300 python bench.py --config $c --no-cpu --path fused > gpurun_out/pbf_$c.json 2> gpurun_out/pbf_$c.err; done
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/pref_C2.json 2> gpurun_out/pref_C2.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_C2.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -c 4 -o gpurun_out/full_C2 python tools/run_conv.py C2 staged 1 > gpurun_out/ncu_full.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_filter -c 1 -o gpurun_out/full_C2_k1 python tools/run_conv.py C2 staged 1 >> gpurun_out/ncu_full.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_fused -c 1 -o gpurun_out/full_C2_fused python tools/run_conv.py C2 fused 1 >> gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
