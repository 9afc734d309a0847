python -m pytest tests/test_gpu_parity.py tests/test_gpu_f3.py tests/test_gpu_f2.py tests/test_gpu_u8.py -x -q -m gpu 2>&1 | tail -2
for cfg in C2 C3 C4; do python tools/time_stage.py $cfg staged 3 50; python tools/time_stage.py $cfg staged 1 50; done
python bench.py --steps 300 --warmup 5 --no-cpu > gpurun_out/probe_C2.json 2>&1; python tools/bench_brief.py gpurun_out/probe_C2.json
