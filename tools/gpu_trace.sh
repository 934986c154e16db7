mkdir -p gpurun_out
FORGE_LIB=dev timeout 300 python tools/probe.py scan > gpurun_out/probe.log 2>&1
FORGE_LIB=dev FORGE_SCAN_NO_TMA_STORE=1 timeout 300 python tools/probe.py scan >> gpurun_out/probe.log 2>&1
FORGE_SCAN_NO_TMA_STORE=1 timeout 120 python tools/trace_scan.py 0 28 >> gpurun_out/trace.log 2>&1
