#!/bin/bash
# A/B the bench over builds ab/<name>.so, alternating: tools/ab_bench.sh A B [rounds]
a=$1; b=$2; n=${3:-2}
for i in $(seq $n); do
  for v in $a $b; do
    echo -n "$v: "; RNSW_DIAG=1 RNSW_LIB=ab/$v.so timeout 300 python bench.py --no-cpu-baseline --no-layer-configs 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], {k: v['ms'] for k, v in d['stages'].items()})"
  done
done
