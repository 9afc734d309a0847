# AUTO's fused c_in limit on C5 (64: layers 4-8 staged, 32: layers 2-8 staged) and C2-C4 staged vs fused
for a in 64 32; do
  WINO_AUTO_FUSED_CIN=$a python bench.py --no-cpu --steps 20 > gpurun_out/am_$a.json 2> gpurun_out/am_$a.err
  echo "== fused c_in <= $a" >> gpurun_out/am.txt
  python tools/brief_r02.py gpurun_out/am_$a.json >> gpurun_out/am.txt 2>&1
done
for c in C2 C3 C4; do for p in fused staged; do
  python bench.py --config $c --path $p --no-cpu --steps 1000 > gpurun_out/am_${c}_$p.json 2> /dev/null
  python tools/brief_r02.py gpurun_out/am_${c}_$p.json >> gpurun_out/am.txt 2>&1
done; done
