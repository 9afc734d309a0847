# ncu --set full captures of the other defaults' GEMM kernels: C3 fused (two 80 KB stages), C4 staged
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_fused -c 1 -o gpurun_out/full_C3_fused python tools/run_conv.py C3 fused 1 > gpurun_out/ncu_c3.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_gemm -c 1 -o gpurun_out/full_C4_staged python tools/run_conv.py C4 staged 1 > gpurun_out/ncu_c4.log 2>&1
ls -la gpurun_out/full_C3_fused.ncu-rep gpurun_out/full_C4_staged.ncu-rep
