for v in k1lag0 k1d16 k1plain; do
  RNSW_DIAG=1 RNSW_LIB=ab/$v.so timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_write.sum,dram__bytes_read.sum --clock-control none -k regex:input_umma -c 3 python tools/one_layer_fused.py conv1_2 256 3 2>/dev/null | grep -E "gpu__time_duration|dram__bytes" | head -6 | sed "s/^/$v /"
done
