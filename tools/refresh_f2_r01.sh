# refresh the fused F(2x2) bench lines and its ncu capture (C2) for profiles/
mkdir -p gpurun_out
for c in C2 C3 C4; do timeout 300 python bench.py --config $c --alg f2 --no-cpu > gpurun_out/f2_${c}.json 2> gpurun_out/f2_${c}.err; done
timeout 300 python bench.py --config C2 --alg f2 --input u8 --no-cpu > gpurun_out/f2u8_C2.json 2> gpurun_out/f2u8_C2.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fused2 -s 3 -c 1 -o gpurun_out/r01_full_C2_f2 \
  python bench.py --no-cpu --config C2 --alg f2 --steps 2 --warmup 3 > gpurun_out/ncu_f2.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r01_launches_C2_f2.csv \
  python bench.py --no-cpu --config C2 --alg f2 --steps 2 --warmup 3 > gpurun_out/ncu_f2_l.log 2>&1
for f in gpurun_out/f2_*.json gpurun_out/f2u8_C2.json; do python tools/bench_brief.py $f; done
