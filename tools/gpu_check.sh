#!/bin/bash
# One GPU round trip: build + smoke, the -m gpu suite, the default bench line.
# usage (under gpurun): bash tools/gpu_check.sh TAG
tag=${1:-run}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1
echo "smoke rc=$?"
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/${tag}_gputest.log 2>&1
echo "gputest rc=$?"; tail -3 gpurun_out/${tag}_gputest.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
echo "bench rc=$?"; cut -c1-400 gpurun_out/${tag}_bench.json
