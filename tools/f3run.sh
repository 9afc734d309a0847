set -x
python -m pytest tests -x -q -m gpu 2>&1 | tail -15 > gpurun_out/f3_tests.log
python bench.py --steps 200 --warmup 5 --no-cpu --target 127 > gpurun_out/f3_bench_C2.json 2> gpurun_out/f3_bench_C2.err
python bench.py --steps 200 --warmup 5 --no-cpu > gpurun_out/f3_bench_C2_255.json 2> gpurun_out/f3_bench_C2_255.err
python bench.py --steps 100 --warmup 5 --no-cpu --target 127 --config C3 > gpurun_out/f3_bench_C3.json 2>&1
cat gpurun_out/f3_tests.log
