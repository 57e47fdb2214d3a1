# K1 (fused gather + sketch) bandwidth evidence on the sketch-heavy variants:
# per-target duration and DRAM traffic under ncu, then the table.
mkdir -p gpurun_out
for c in ${K1_CONFIGS-c4a20 c5s64k}; do
  timeout 900 python tools/k1_probe.py $c > gpurun_out/k1_probe_$c.log 2> gpurun_out/k1_probe_$c.err
  echo "probe $c exit=$?"
  timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum \
    --clock-control none -k regex:sketch --csv --log-file gpurun_out/k1_ncu_$c.csv python tools/k1_probe.py $c > gpurun_out/k1_ncu_$c.log 2>&1
  echo "ncu $c exit=$?"
  python tools/k1_table.py gpurun_out/k1_ncu_$c.csv gpurun_out/k1_ncu_$c.log > gpurun_out/k1_table_$c.txt 2>&1
  cat gpurun_out/k1_table_$c.txt
done
