# refresh the uint8 (f2 row) fused bench lines for profiles/
for c in C2 C3; do timeout 300 python bench.py --config $c --input u8 --no-cpu > gpurun_out/u8_${c}.json 2> gpurun_out/u8_${c}.err; python tools/bench_brief.py gpurun_out/u8_${c}.json | head -1; done
