# usage: bash tools/gpu_stage_ab.sh <stage> "<variants>"  -- per-layer stage ms of each variant (no tests)
for v in $2; do
  echo -n "$v: "; RNSW_DIAG=1 RNSW_LIB=ab/$v.so timeout 300 python bench.py --no-cpu-baseline --no-layer-configs --steps 5 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['stages']['$1']['ms'], [v.get('$1') for v in d['config']['layer_stage_ms'].values()])"
done
