mkdir -p gpurun_out
for R in 1 9 1 9; do echo "ring=$R" >> gpurun_out/prefetch.log; FORGE_LIB=dev FORGE_SCAN_RING=$R timeout 300 python tools/probe.py scan >> gpurun_out/prefetch.log 2>&1; done
for op in 0 11; do FORGE_SCAN_RING=1 timeout 120 python tools/trace_lag.py $op 28 >> gpurun_out/prefetch.log 2>&1; done
exit 0
