mkdir -p gpurun_out; : > gpurun_out/exp_r.log
FORGE_SCAN_SUBTILES=2 timeout 300 python tools/probe.py scan --check >> gpurun_out/exp_r.log 2>&1
FORGE_SCAN_SUBTILES=1 timeout 300 python tools/probe.py scan >> gpurun_out/exp_r.log 2>&1
FORGE_SCAN_SUBTILES=2 FORGE_SCAN_LOOKBACK=99 timeout 300 python tools/probe.py scan >> gpurun_out/exp_r.log 2>&1
FORGE_SCAN_SUBTILES=2 timeout 300 python tools/trace_scan.py 0 28 2>&1 | grep -v "^  \|^ }" >> gpurun_out/exp_r.log 2>&1
