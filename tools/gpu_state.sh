# state check: GPU tests, default bench line, smoke
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/st_smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/st_gputest.log 2>&1; echo "gputest rc=$?"; tail -4 gpurun_out/st_gputest.log
timeout 600 python bench.py > gpurun_out/st_bench.json 2> gpurun_out/st_bench.err; echo "bench rc=$?"; tail -c 3000 gpurun_out/st_bench.json
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/st_smoke.log 2>&1; echo "smoke rc=$?"
