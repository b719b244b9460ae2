timeout 300 python tools/one_layer_fused.py conv1_2 64 2 > gpurun_out/o_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:output_kron -s 1 -c 1 -o gpurun_out/k4k2_conv1_2_b64 python tools/one_layer_fused.py conv1_2 64 2 > gpurun_out/o_ncu.log 2>&1; echo "ncu rc=$?"
