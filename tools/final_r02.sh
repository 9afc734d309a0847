# round-2 final measurements: GPU tests + smoke, the default bench (C5) and C2-C4 lines with the CPU baseline,
# the reference (oracle) arm, the C5 launch list (ncu, after the plain run exited 0)
set -o pipefail
mkdir -p gpurun_out/final
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3 > gpurun_out/final/tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/final/smoke.txt
timeout 900 python bench.py > gpurun_out/final/r02_bench_C5.json 2> gpurun_out/final/r02_bench_C5.err
for c in C2 C3 C4; do timeout 600 python bench.py --config $c > gpurun_out/final/r02_bench_$c.json 2> gpurun_out/final/r02_bench_$c.err; done
timeout 600 python bench.py --impl reference --steps 13 --warmup 3 > gpurun_out/final/r02_reference_C5.json 2> gpurun_out/final/r02_reference_C5.err
python tools/run_c5_r02.py step 1 > gpurun_out/final/plain_step.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final/r02_launches_C5.csv \
  python tools/run_c5_r02.py step 1 > gpurun_out/final/ncu_step.log 2>&1
python tools/brief_r02.py gpurun_out/final/r02_bench_C*.json > gpurun_out/final/brief.txt 2>&1
