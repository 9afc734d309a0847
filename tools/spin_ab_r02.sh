# A/B of the barrier-wait flavour in K3F (suspending try_wait vs test_wait spin) for the MMA issuer and the
# epilogue handshake: C2-C4 bench lines + C5 per-layer kernel times per variant; default build restored at the end
set -o pipefail
python -m pytest tests -m gpu -x -q 2>&1 | tail -2 > gpurun_out/spin_tests.txt
for v in base mma epi both; do
  case $v in base) f="";; mma) f="-DWINO_SPIN_MMA";; epi) f="-DWINO_SPIN_EPI";; both) f="-DWINO_SPIN_MMA -DWINO_SPIN_EPI";; esac
  WINO_NVCC_FLAGS="$f" python -c "from paper_1901_01965_b200 import build as B; B.build(force=True)" > /dev/null 2>&1 || exit 1
  for c in C2 C3 C4; do python bench.py --config $c --no-cpu --steps 1000 > gpurun_out/s_${v}_$c.json 2> /dev/null; done
  python tools/c5_layers_r02.py > gpurun_out/s_${v}_c5l.txt 2>&1
  echo "== $v" >> gpurun_out/spin.txt
  python tools/brief_r02.py gpurun_out/s_${v}_C2.json gpurun_out/s_${v}_C3.json gpurun_out/s_${v}_C4.json >> gpurun_out/spin.txt 2>&1
  grep "whole step\|layer  [12]:" gpurun_out/s_${v}_c5l.txt >> gpurun_out/spin.txt
done
