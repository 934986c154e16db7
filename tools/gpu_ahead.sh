mkdir -p gpurun_out
for P in 100 200 300 400 200 300; do echo "ahead=$P" >> gpurun_out/ahead.log; FORGE_LIB=dev FORGE_SCAN_PREFETCH_AHEAD=$P timeout 300 python tools/probe.py scan >> gpurun_out/ahead.log 2>&1; done
exit 0
