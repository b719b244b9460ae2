# usage: bash tools/gpu_unfused_ab.sh "<variants>" [rounds] -- int32-output (unfused) stack: per-stage ms per variant, after the GPU tests of the in-tree build
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/ab_gputest.log 2>&1; echo "gputest rc=$?"; tail -2 gpurun_out/ab_gputest.log
n=${2:-2}
for b in 256 32; do for i in $(seq $n); do
  for v in $1; do
    echo -n "b$b $v: "; RNSW_DIAG=1 RNSW_LIB=ab/$v.so timeout 300 python bench.py --unfused --batch $b --no-cpu-baseline --no-layer-configs 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], {k: v['ms'] for k, v in d['stages'].items()}, d['clocks']['sm_mhz'])"
  done
done; done
