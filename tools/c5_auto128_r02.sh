# GPU tests (K2 refactor) + C5 with AUTO's fused c_in limit 256 (default) vs 128 (layers 6-8 staged)
set -o pipefail
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2 > gpurun_out/a128_tests.txt
for a in 256 128; do
  WINO_AUTO_FUSED_CIN=$a python bench.py --no-cpu --steps 20 > gpurun_out/a128_$a.json 2> gpurun_out/a128_$a.err
  echo "== fused c_in <= $a" >> gpurun_out/a128.txt
  python tools/brief_r02.py gpurun_out/a128_$a.json >> gpurun_out/a128.txt 2>&1
done
