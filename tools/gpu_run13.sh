for b in 1 32; do
timeout 300 python bench.py --steps 20 --warmup 5 --batch $b --no-cpu-baseline --no-layer-configs > gpurun_out/p_bench_b$b.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/p_bench_b$b.json'))
print($b, d['value'], d['ms_per_step'], d['e2e']['value']); print({k:(v['ms'],v.get('GB_s')) for k,v in d['stages'].items()}); print({k:v for k,v in d['config']['layer_stage_ms'].items()})"
done
