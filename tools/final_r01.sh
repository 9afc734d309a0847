# full GPU test suite + smoke + default bench (what the driver runs at round end), with timeouts
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/final_C2.json 2> gpurun_out/final_C2.err; python tools/bench_brief.py gpurun_out/final_C2.json
