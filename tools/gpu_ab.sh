# usage: bash tools/gpu_ab.sh "<variant names>" [rounds]  -- GPU tests on the in-tree build, then A/B benches
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/ab_gputest.log 2>&1; echo "gputest rc=$?"; tail -3 gpurun_out/ab_gputest.log
n=${2:-2}
for i in $(seq $n); do
  for v in $1; do
    echo -n "$v: "; RNSW_DIAG=1 RNSW_LIB=ab/$v.so timeout 300 python bench.py --no-cpu-baseline --no-layer-configs 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], {k: v['ms'] for k, v in d['stages'].items()}, d['clocks']['sm_mhz'])"
  done
done
