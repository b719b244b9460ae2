# one-rank check of the multi-rank code path: NCCL init, gather and max-over-ranks as real collectives
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_gemm_t.py -m gpu -x -q -p no:cacheprovider > gpurun_out/gemmt_test.log 2>&1; echo "gemmt test rc=$?"; tail -2 gpurun_out/gemmt_test.log
RNSW_BENCH_FORCE_DIST=1 NCCL_DEBUG=INFO timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 \
  bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu-baseline --no-layer-configs > gpurun_out/dist1.json 2> gpurun_out/dist1.err; echo "dist1 rc=$?"
python - <<'P'
import json
d=json.loads([l for l in open('gpurun_out/dist1.json') if l.startswith('{')][-1])
print({k:d[k] for k in ('value','ms_per_step','n_gpus','scaling')}, d['e2e']['value'], d.get('forced_collectives'))
P
grep -c "NCCL INFO" gpurun_out/dist1.json gpurun_out/dist1.err; grep -m3 "NCCL INFO.*\(comm\|Init\)" gpurun_out/dist1.json gpurun_out/dist1.err | cut -c1-200
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29518 \
  bench.py --impl reference --gpus 1 --steps 1 --warmup 0 > gpurun_out/ref1.json 2> gpurun_out/ref1.err; echo "ref rc=$?"; tail -c 600 gpurun_out/ref1.json
