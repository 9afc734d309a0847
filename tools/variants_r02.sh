# r02 refresh of the SURVEY 8(f) variant lines: F(2x2) (--alg f2), uint8 (--input u8), int8-native target (--target 127)
for c in C2 C3 C4; do
  python bench.py --config $c --alg f2 --no-cpu > gpurun_out/v_${c}_f2.json 2>/dev/null; echo "f2 $(python tools/brief_r02.py gpurun_out/v_${c}_f2.json | head -1 | cut -d' ' -f1-4)"
  python bench.py --config $c --input u8 --no-cpu > gpurun_out/v_${c}_u8.json 2>/dev/null; echo "u8 $(python tools/brief_r02.py gpurun_out/v_${c}_u8.json | head -1 | cut -d' ' -f1-4)"
  python bench.py --config $c --target 127 --path staged --no-cpu > gpurun_out/v_${c}_f3.json 2>/dev/null; echo "f3 $(python tools/brief_r02.py gpurun_out/v_${c}_f3.json | head -1 | cut -d' ' -f1-4)"
done
python bench.py --config C2 --alg f2 --input u8 --no-cpu > gpurun_out/v_C2_f2u8.json 2>/dev/null; echo "f2u8 $(python tools/brief_r02.py gpurun_out/v_C2_f2u8.json | head -1 | cut -d' ' -f1-4)"
