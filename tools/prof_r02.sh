# r02 profiles: launch list of one C5 step; ncu --set full of layer 2's fused GEMM (the C5 dominant kernel)
python tools/run_c5_r02.py step 1 > gpurun_out/plain_step.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_C5.csv \
    python tools/run_c5_r02.py step 1 > gpurun_out/ncu_step.log 2>&1
python tools/run_c5_r02.py layer 2 2 > gpurun_out/plain_l2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_fused -s 20 -c 1 -o gpurun_out/r02_full_C5_L2_fused \
    python tools/run_c5_r02.py layer 2 2 > gpurun_out/ncu_l2.log 2>&1
