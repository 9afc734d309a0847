# ncu --set full of C5 layer 1's fused GEMM (quarter-K packing, c_in = 3)
python tools/run_c5_r02.py layer 1 2 > gpurun_out/plain_l1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_fused -s 30 -c 1 -f -o gpurun_out/r02_full_C5_L1_fused \
    python tools/run_c5_r02.py layer 1 2 > gpurun_out/ncu_l1.log 2>&1
