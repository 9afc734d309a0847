# K3 probe: parity of the staged path, stage-3 timings under WINO_K3_DBG modes, a short C2 bench
python -m pytest tests/test_gpu_parity.py tests/test_gpu_f3.py tests/test_gpu_f2.py -x -q -m gpu 2>&1 | tail -3
for cfg in C2 C4; do
  for d in 0 1 2 14; do
    WINO_K3_DBG=$d python tools/time_stage.py $cfg staged 3 50 | sed "s/^/dbg=$d /"
  done
done
python bench.py --steps 300 --warmup 5 --no-cpu > gpurun_out/probe_C2.json 2>&1; python tools/bench_brief.py gpurun_out/probe_C2.json 2>/dev/null || tail -c 600 gpurun_out/probe_C2.json
