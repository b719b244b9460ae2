# A/B the fused stack: RNSW_LIB=ab/A.so vs ab/B.so, alternating, 3 rounds
for i in 1 2; do
  for v in A B; do
    echo -n "$v: "; RNSW_DIAG=1 RNSW_LIB=ab/$v.so python tools/probe_vgg.py 256 2>&1 | grep "fused total"
  done
done
