timeout 300 python tools/one_layer.py conv1_2 64 2 > gpurun_out/j_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:output_umma -s 1 -c 1 -o gpurun_out/k4_r2_conv1_2_b64 python tools/one_layer.py conv1_2 64 2 > gpurun_out/j_ncu.log 2>&1; echo "ncu rc=$?"
timeout 300 python tools/one_layer.py conv1_2 64 2 > gpurun_out/j_plain2.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:winograd_gemm -s 1 -c 1 -o gpurun_out/gemm_r2_conv1_2_b64 python tools/one_layer.py conv1_2 64 2 > gpurun_out/j_ncu2.log 2>&1; echo "ncu rc=$?"
