timeout 300 python tools/one_layer_fused.py conv1_1 256 2 > gpurun_out/p_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:smallc -s 1 -c 1 \
  -o gpurun_out/r02c_smallc_conv1_1_b256 python tools/one_layer_fused.py conv1_1 256 2 > gpurun_out/p_ncu.log 2>&1; echo "rc=$?"
python tools/ncu_summary.py gpurun_out/r02c_smallc_conv1_1_b256.ncu-rep > gpurun_out/p_sum.txt 2>&1
ncu -i gpurun_out/r02c_smallc_conv1_1_b256.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
rows=list(csv.reader(sys.stdin)); hdr=rows[0]; vals=rows[2]
for h,v in zip(hdr,vals):
    if any(k in h for k in ['dram__throughput','lts__throughput','l1tex__throughput','sm__throughput','achieved_occupancy','warps_active','lts__t_sectors_op_write','dram__bytes_write.sum','dram__bytes_read.sum','lts__t_sectors_srcunit_tex_op_write','smsp__issue_active']): print(h, v)
" >> gpurun_out/p_sum.txt
