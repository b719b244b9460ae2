# usage: bash tools/gpu_cfg_ab.sh "<variants>"  -- BASELINE configs 1/3/5 device latencies per variant
for v in $1; do
  echo -n "$v: "; RNSW_DIAG=1 RNSW_LIB=ab/$v.so timeout 300 python tools/cfg_lat.py 2>/dev/null | tail -1
done
