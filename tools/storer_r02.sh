# HISTORICAL: the experiment switch this script exercises was removed after the measurement (not kept;
# DESIGN.md 6b records the result); kept to document how the numbers in profiles/ were taken.
# storer-warp K3F: GPU tests, C2-C5 lines, C5 per-layer times
set -o pipefail
bash tools/quick_r02.sh
python tools/c5_layers_r02.py > gpurun_out/c5l.txt 2>&1
grep "whole step\|layer  [0-9]:\|layer 1[0-3]:" gpurun_out/c5l.txt | cut -c1-60 >> gpurun_out/quick.txt
