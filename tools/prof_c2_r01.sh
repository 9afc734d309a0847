# profile refresh for the default C2 path (fused) and C5 after kernel changes
timeout 600 python bench.py --config C2 > gpurun_out/pb_C2.json 2> gpurun_out/pb_C2.err
timeout 900 python bench.py --config C5 --no-cpu > gpurun_out/pb_C5.json 2> gpurun_out/pb_C5.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_C2.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_launch.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -c 4 -o gpurun_out/full_C2_fused python tools/run_conv.py C2 fused 1 > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out/full_C2_fused.ncu-rep gpurun_out/launches_C2.csv
