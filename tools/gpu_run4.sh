mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r_gputest.log 2>&1; echo "gputest rc=$?"; tail -4 gpurun_out/r_gputest.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-layer-configs > gpurun_out/r_bench.json 2> gpurun_out/r_bench.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/r_bench.json'))
print(d['value'], d['ms_per_step']); print({k:(v['ms'],v['GB_s']) for k,v in d['stages'].items()}); print({k:v.get('input_transform') for k,v in d['config']['layer_stage_ms'].items()})"
timeout 300 python tools/one_layer_fused.py conv1_2 64 2 > gpurun_out/r_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:output_umma -s 1 -c 1 -o gpurun_out/k4u_r2_conv1_2_b64 python tools/one_layer_fused.py conv1_2 64 2 > gpurun_out/r_ncu.log 2>&1; echo "ncu rc=$?"
