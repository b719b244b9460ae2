#!/bin/bash
# A/B the input transform stage over diagnostic builds ab/<name>.so
for v in "$@"; do
  for L in conv1_2 conv2_2 conv3_2; do
    echo -n "$v: "; RNSW_DIAG=1 RNSW_LIB=ab/$v.so timeout 120 python tools/time_k1.py $L 256 10 2>/dev/null
  done
done
