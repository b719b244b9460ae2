timeout 300 python tools/kron_probe.py
timeout 900 python -m pytest tests/test_gpu_kron.py tests/test_gpu_configs.py -x -q -p no:cacheprovider > gpurun_out/n_kron.log 2>&1; echo "kron rc=$?"; tail -3 gpurun_out/n_kron.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-layer-configs > gpurun_out/n_bench.json 2> gpurun_out/n_bench.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/n_bench.json'))
print(d['value'], d['ms_per_step']); print({k:(v['ms'],v['GB_s']) for k,v in d['stages'].items()}); print({k:v.get('output_transform') for k,v in d['config']['layer_stage_ms'].items()})"
