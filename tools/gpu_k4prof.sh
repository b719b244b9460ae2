mkdir -p gpurun_out
timeout 300 python tools/one_layer_fused.py conv1_2 64 2 > gpurun_out/k4p_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:output_umma -s 1 -c 1 \
  -o gpurun_out/k4p_conv1_2_b64 python tools/one_layer_fused.py conv1_2 64 2 > gpurun_out/k4p_ncu.log 2>&1; echo "k4 rc=$?"
python tools/ncu_stalls.py gpurun_out/k4p_conv1_2_b64.ncu-rep 60 > gpurun_out/k4p_stalls.txt 2>&1
python tools/ncu_summary.py gpurun_out/k4p_conv1_2_b64.ncu-rep > gpurun_out/k4p_summary.txt 2>&1
