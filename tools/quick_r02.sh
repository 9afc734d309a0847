# GPU tests + short bench lines for C2-C5 (no CPU baseline); summary in gpurun_out/quick.txt
set -o pipefail
python -m pytest tests -m gpu -x -q 2>&1 | tail -2 > gpurun_out/quick_tests.txt
for c in C2 C3 C4; do python bench.py --config $c --no-cpu --steps 1000 > gpurun_out/q_$c.json 2> gpurun_out/q_$c.err; done
python bench.py --no-cpu --steps 20 > gpurun_out/q_C5.json 2> gpurun_out/q_C5.err
python tools/brief_r02.py gpurun_out/q_C2.json gpurun_out/q_C3.json gpurun_out/q_C4.json gpurun_out/q_C5.json > gpurun_out/quick.txt 2>&1
cat gpurun_out/quick_tests.txt >> gpurun_out/quick.txt
