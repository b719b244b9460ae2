# round-2 (final session) evidence: GPU tests, bench lines, per-launch list of one
# fused VGG16 step at batch 256 (time + DRAM bytes), full ncu captures of K1 and K4
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/f_gputest.log 2>&1; echo "gputest rc=$?"; tail -2 gpurun_out/f_gputest.log
timeout 600 python bench.py > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err; echo "bench rc=$?"
for b in 1 32; do timeout 300 python bench.py --batch $b --no-cpu-baseline --no-layer-configs > gpurun_out/f_bench_b$b.json 2>/dev/null; echo "bench b$b rc=$?"; done
timeout 300 python tools/stack_once.py 256 > gpurun_out/f_s_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/r02d_launches.csv python tools/stack_once.py 256 > gpurun_out/f_ncu1.log 2>&1; echo "launches rc=$?"
timeout 300 python tools/one_layer_fused.py conv1_2 256 2 > gpurun_out/f_plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:input_umma -s 1 -c 1 \
  -o gpurun_out/r02d_k1u_conv1_2_b256 python tools/one_layer_fused.py conv1_2 256 2 > gpurun_out/f_ncu2.log 2>&1; echo "k1u rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:output_umma -s 1 -c 1 \
  -o gpurun_out/r02d_k4umma_conv1_2_b256 python tools/one_layer_fused.py conv1_2 256 2 > gpurun_out/f_ncu3.log 2>&1; echo "k4 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:winograd_gemm -s 1 -c 1 \
  -o gpurun_out/r02d_gemm_conv3_2_b256 python tools/one_layer_fused.py conv3_2 256 2 > gpurun_out/f_ncu4.log 2>&1; echo "gemm rc=$?"
