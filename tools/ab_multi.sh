# bench value per variant .so in ab/ (names as args), two rounds
for i in 1 2; do
  for v in "$@"; do
    echo -n "$v: "; RNSW_DIAG=1 RNSW_LIB=ab/$v.so python bench.py --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], {k: v['ms'] for k, v in d['stages'].items()})"
  done
done
