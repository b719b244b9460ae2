# round-2 evidence: per-launch list (time + DRAM bytes) of one fused VGG16 step
# at batch 256, and full ncu captures of the K1 / GEMM kernels on conv layers
mkdir -p gpurun_out
timeout 300 python tools/stack_once.py 256 > gpurun_out/s_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/r02_launches.csv python tools/stack_once.py 256 > gpurun_out/s_ncu1.log 2>&1; echo "launches rc=$?"
timeout 300 python tools/one_layer_fused.py conv1_2 256 2 > gpurun_out/s_plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:input_umma -s 1 -c 1 \
  -o gpurun_out/r02_k1u_conv1_2_b256 python tools/one_layer_fused.py conv1_2 256 2 > gpurun_out/s_ncu2.log 2>&1; echo "k1u rc=$?"
timeout 300 python tools/one_layer_fused.py conv3_2 256 2 > gpurun_out/s_plain3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:winograd_gemm -s 1 -c 1 \
  -o gpurun_out/r02_gemm_conv3_2_b256 python tools/one_layer_fused.py conv3_2 256 2 > gpurun_out/s_ncu3.log 2>&1; echo "gemm rc=$?"
