timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/q_gputest.log 2>&1; echo "gputest rc=$?"; tail -4 gpurun_out/q_gputest.log
for b in 1 32 256; do
timeout 300 python bench.py --steps 10 --warmup 3 --batch $b --no-cpu-baseline --no-layer-configs > gpurun_out/q_bench_b$b.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/q_bench_b$b.json'))
print($b, d['value'], d['ms_per_step']); print({k:(v['ms'],v.get('GB_s')) for k,v in d['stages'].items()})"
done
