# A/B the bench value: RNSW_LIB=ab/A.so vs ab/B.so, alternating
for i in 1 2; do
  for v in A B; do
    echo -n "$v: "; RNSW_DIAG=1 RNSW_LIB=ab/$v.so python bench.py --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], {k: v['ms'] for k, v in d['stages'].items()}); print('   out/layer', [v.get('output_transform') for v in d['config']['layer_stage_ms'].values()])"
  done
done
