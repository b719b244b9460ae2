# per-layer gemm ms for variant .so files (names as args); bench does no correctness check
for v in "$@"; do
  echo -n "$v: "; RNSW_DIAG=1 RNSW_LIB=ab/$v.so python bench.py --no-cpu-baseline --steps 5 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], [v.get('gemm') for v in d['config']['layer_stage_ms'].values()])"
done
