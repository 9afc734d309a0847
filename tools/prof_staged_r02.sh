# ncu --set full of the staged GEMM (k_gemm) on C5 layers 6 (c_in 256) and 9 (c_in 512), after plain runs
for L in 6 9; do
  python tools/run_c5_r02.py layer $L 2 > gpurun_out/plain_l$L.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_gemm -s 47 -c 1 -o gpurun_out/r02_full_C5_L${L}_gemm \
      python tools/run_c5_r02.py layer $L 2 > gpurun_out/ncu_l$L.log 2>&1
done
