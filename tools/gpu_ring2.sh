# ring variants (FORGE_SCAN_RING bits: 1 discard, 2 evict_last stores), trace, DRAM bytes (development)
mkdir -p gpurun_out
for R in 0 1 2 3; do
  echo "ring=$R" >> gpurun_out/ring2.log
  FORGE_LIB=dev FORGE_SCAN_RING=$R timeout 300 python tools/probe.py scan >> gpurun_out/ring2.log 2>&1
done
for op in 0 10 11; do
  FORGE_SCAN_RING=1 timeout 120 python tools/trace_lag.py $op 28 >> gpurun_out/ring2_trace.log 2>&1
done
for R in 0 1 2; do for op in 0 10; do
  FORGE_LIB=dev FORGE_SCAN_RING=$R timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:scan_lag -s 2 -c 1 --csv python tools/one_kernel.py scan $op > gpurun_out/ring2_ncu_${R}_${op}.csv 2>&1
done; done
