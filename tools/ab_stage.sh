# per-layer stage ms (arg1 = stage kind) for variant .so files (rest of args)
kind=$1; shift
for v in "$@"; do
  echo -n "$v: "; RNSW_DIAG=1 RNSW_LIB=ab/$v.so python bench.py --no-cpu-baseline --no-layer-configs --steps 5 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], [v.get('$kind') for v in d['config']['layer_stage_ms'].values()])"
done
