# usage: bash tools/gpu_gemmt_ab.sh  -- small-P GEMM range sweep at batch 32 / 64 / 8 (stage and per-layer GEMM times)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemm_t.py -m gpu -x -q -p no:cacheprovider > gpurun_out/gemmt_test.log 2>&1; echo "gemmt test rc=$?"; tail -3 gpurun_out/gemmt_test.log
for b in 32 64 8; do
  for mp in 48 64 96 128; do
    echo -n "b$b T=$mp: "; RNSW_GEMM_T=$mp timeout 300 python bench.py --batch $b --no-cpu-baseline --no-layer-configs 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], {k: v['ms'] for k, v in d['stages'].items()}, [v.get('gemm') for v in d['config']['layer_stage_ms'].values()])"
  done
done
