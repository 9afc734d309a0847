for cfg in C2 C4; do python tools/time_stage.py $cfg staged 3 50; done
python bench.py --steps 300 --warmup 5 --no-cpu > gpurun_out/probe_C2.json 2>&1; python tools/bench_brief.py gpurun_out/probe_C2.json
