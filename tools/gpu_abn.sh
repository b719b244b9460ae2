# usage: bash tools/gpu_abn.sh "<variants>" [rounds]  -- A/B benches only, alternating
n=${2:-3}
for i in $(seq $n); do
  for v in $1; do
    echo -n "$v: "; RNSW_DIAG=1 RNSW_LIB=ab/$v.so timeout 300 python bench.py --no-cpu-baseline --no-layer-configs 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], {k: v['ms'] for k, v in d['stages'].items()}, d['clocks']['sm_mhz'])"
  done
done
