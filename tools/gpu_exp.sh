# Scratch GPU experiment (development; overwritten per experiment)
mkdir -p gpurun_out; : > gpurun_out/exp.log
FORGE_SCAN_LOOKBACK=3 timeout 300 python tools/probe.py scan --check | sed "s/^/groups /" >> gpurun_out/exp.log 2>&1
timeout 300 python tools/probe.py scan | sed "s/^/flat /" >> gpurun_out/exp.log 2>&1
FORGE_SCAN_LOOKBACK=3 timeout 300 python tools/trace_scan.py 0 28 2>&1 | grep -v "^  \|^ }" | sed "s/^/groups trace /" >> gpurun_out/exp.log 2>&1
