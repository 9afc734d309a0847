# C1 at 8 ranks (4 empty Cout shards) in the gloo validation mode, with per-rank progress
export WINO_DIST_BACKEND=gloo WINO_BENCH_TRACE=1
timeout 900 python bench.py --gpus 8 --config C1 --steps 20 --warmup 3 --no-cpu > gpurun_out/mr_C1x8.json 2> gpurun_out/mr_C1x8.err; echo "C1 x8 rc=$?"
timeout 300 python bench.py --gpus 2 --config C1 --steps 20 --warmup 3 --no-cpu > gpurun_out/mr_C1x2.json 2> gpurun_out/mr_C1x2.err; echo "C1 x2 rc=$?"
grep "^\[rank" gpurun_out/mr_C1x8.err | tail -40
tail -c 600 gpurun_out/mr_C1x8.json; tail -c 600 gpurun_out/mr_C1x2.json
