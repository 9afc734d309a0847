# final ncu --set full captures: C5 layer 2's input transform (four slices per CTA) and fused GEMM
python tools/run_c5_r02.py layer 2 2 > gpurun_out/plain_l2f.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_input_transform_f4 -s 30 -c 1 -o gpurun_out/r02_full_C5_L2_k2 \
    python tools/run_c5_r02.py layer 2 2 > gpurun_out/ncu_l2k2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_fused -s 30 -c 1 -o gpurun_out/r02_full_C5_L2_fused_final \
    python tools/run_c5_r02.py layer 2 2 > gpurun_out/ncu_l2kf.log 2>&1
