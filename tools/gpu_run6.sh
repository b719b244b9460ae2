RNSW_DIAG=1 RNSW_LIB=ab/k1p1.so timeout 120 python tools/time_k1.py conv1_2 64 3 > gpurun_out/h_plain.log 2>&1 && \
RNSW_DIAG=1 RNSW_LIB=ab/k1p1.so timeout 600 ncu --set full --clock-control none --import-source on -k regex:input_umma -s 2 -c 1 -o gpurun_out/k1p1_conv1_2_b64 python tools/time_k1.py conv1_2 64 3 > gpurun_out/h_ncu.log 2>&1; echo "ncu rc=$?"
timeout 120 python tools/time_k1.py conv1_2 64 3 > gpurun_out/h_plain0.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:input_umma -s 2 -c 1 -o gpurun_out/k1p0_conv1_2_b64 python tools/time_k1.py conv1_2 64 3 > gpurun_out/h_ncu0.log 2>&1; echo "ncu rc=$?"
