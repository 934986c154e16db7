mkdir -p gpurun_out
timeout 300 python tools/probe.py scan --check > gpurun_out/ring9.log 2>&1
for R in 1 0 3; do
  echo "ring=$R" >> gpurun_out/ring9.log
  FORGE_LIB=dev FORGE_SCAN_RING=$R timeout 120 python tools/probe.py scan >> gpurun_out/ring9.log 2>&1
done
for op in 12 10 0; do timeout 60 python tools/hang_probe.py $op 300 27 >> gpurun_out/ring9.log 2>&1; done
timeout 120 python tools/hang_probe2.py 40 28 >> gpurun_out/ring9.log 2>&1
for op in 0 10 11; do
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:scan_lag -s 2 -c 1 --csv python tools/one_kernel.py scan $op > gpurun_out/ring9_ncu_${op}.csv 2>&1
done
timeout 1500 python -m pytest tests -m gpu -q -x -k "lag or stress or scan" -p no:randomly > gpurun_out/pytest_ring9.log 2>&1; echo rc=$? >> gpurun_out/pytest_ring9.log
exit 0
