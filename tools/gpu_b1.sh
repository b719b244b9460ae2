# batch-1 (BASELINE config 2) bench line summary
python bench.py --batch 1 --steps 50 --warmup 10 --no-cpu-baseline > gpurun_out/b1.jsonl 2>&1
python -c "
import json;d=json.loads(open('gpurun_out/b1.jsonl').read().strip().splitlines()[-1]);print('b1', d['value'],d['ms_per_step'],{k: v['ms'] for k, v in d['stages'].items()})"
