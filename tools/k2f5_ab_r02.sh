# HISTORICAL: the experiment switch this script exercises was removed after the measurement (not kept;
# DESIGN.md 6b records the result); kept to document how the numbers in profiles/ were taken.
# pipelined K2F (cp.async into a per-thread slot refilled after the column transform, WINO_K2F5=1) vs the
# current K2F: GPU parity with it on, stage-2 times at C2/C4 and C2-shaped batches 32/128/512, C5 lines
set -o pipefail
WINO_K2F5=1 timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2 > gpurun_out/f5_tests.txt
for f in "0 50" "1 50" "1 0"; do
  set -- $f
  echo "== K2F5=$1 carve=$2" >> gpurun_out/f5.txt
  for c in C2 C4; do WINO_K2F5=$1 WINO_K2F5_CARVE=$2 python tools/time_stage.py $c fused 2 50 >> gpurun_out/f5.txt 2>&1; done
  for n in 32 128 512; do WINO_K2F5=$1 WINO_K2F5_CARVE=$2 python tools/k2_ablate_r02.py $n >> gpurun_out/f5.txt 2>&1; done
done
for f in 0 1; do
  WINO_K2F5=$f python bench.py --no-cpu --steps 20 > gpurun_out/f5_C5_$f.json 2> gpurun_out/f5_C5_$f.err
  python tools/brief_r02.py gpurun_out/f5_C5_$f.json >> gpurun_out/f5.txt 2>&1
done
